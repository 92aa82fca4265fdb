// rs_device.cuh — sm_100a device primitives for the region-streaming runtime.
//
// Warp-synchronous helpers (ballot/popc compaction, shuffles), TMA bulk
// copies (cp.async.bulk global->shared with an mbarrier transaction count),
// mbarrier waits, and the aggregate traits (begin/run/end of Fig. 5,
// PAPER.md P:532-534) used by the persistent pipeline kernel in rs.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rs {

constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint32_t lanemask_le() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

// 32-bit shared-window addressing (one LEA forms a compaction store address;
// immediate offsets fold a slice's 128-byte stride into the load)
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// a * 4 + b as one opaque step (one LEA)
__device__ __forceinline__ uint32_t lea4(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// Non-blocking probe: has the phase with the given parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Potentially-suspending probe (hardware sleep up to a system time limit).
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Warp-uniform probe: lane 0 tests the phase, the verdict is broadcast and
// __syncwarp carries lane 0's acquire to the other lanes.  (Per-lane probes
// can disagree when the phase completes while the instruction executes.)
__device__ __forceinline__ bool mbar_test_uniform(uint64_t *bar, uint32_t parity) {
    bool ok = false;
    if ((threadIdx.x & 31u) == 0) ok = mbar_test(bar, parity);
    ok = __shfl_sync(kFull, (int)ok, 0) != 0;
    __syncwarp();
    return ok;
}
__device__ __forceinline__ bool mbar_try_wait_uniform(uint64_t *bar, uint32_t parity) {
    bool ok = false;
    if ((threadIdx.x & 31u) == 0) ok = mbar_try_wait(bar, parity);
    ok = __shfl_sync(kFull, (int)ok, 0) != 0;
    __syncwarp();
    return ok;
}

// ------------------------------------------------------------- TMA (bulk)
// 1-D bulk copy global -> shared, completion signalled on `bar` as tx bytes.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
// Order this thread's earlier generic-proxy shared accesses before later
// async-proxy (TMA) writes to the same buffer (ring-slot reuse).
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// --------------------------------------------------------- aggregate traits
// begin() = identity, run() = combine(lift(v)), end() = store (Fig. 5,
// P:532-534).  Identities per DESIGN.md reading A1.
template <int AGG>
struct AggT;

template <>
struct AggT<20> {  // RS_OP_SUM_I64 over int32 elements
    static constexpr bool heavy = false;   // lift costs far more than a select (fused paths lift survivors only)
    static constexpr bool group = true;    // exact inverse: segment sums as prefix differences
    __device__ static unsigned long long sub(unsigned long long a, unsigned long long b) { return a - b; }
    using A = unsigned long long;  // two's-complement wraparound sum
    __device__ static A id() { return 0ull; }
    __device__ static A lift(uint32_t v) { return (A)(long long)(int)v; }
    __device__ static A lift_i(uint32_t v, long long) { return lift(v); }
    __device__ static A comb(A a, A b) { return a + b; }
    __device__ static A shfl(A a, int src) { return __shfl_sync(kFull, a, src); }
    __device__ static A shfl_up(A a, int d) { return __shfl_up_sync(kFull, a, d); }
    __device__ static A shfl_xor(A a, int m) { return __shfl_xor_sync(kFull, a, m); }
    __device__ static void store(void *o0, void *, uint64_t i, A a) { ((A *)o0)[i] = a; }
    __device__ static A load(const void *o0, const void *, uint64_t i) { return ((const A *)o0)[i]; }
    static constexpr int bytes0 = 8, bytes1 = 0;
};

template <>
struct AggT<21> {  // RS_OP_SUM_F32 over fp32 elements
    static constexpr bool heavy = false;   // lift costs far more than a select (fused paths lift survivors only)
    static constexpr bool group = false;   // fp32: prefix differences would cancel
    using A = float;
    __device__ static A id() { return 0.0f; }
    __device__ static A lift(uint32_t v) { return __uint_as_float(v); }
    __device__ static A lift_i(uint32_t v, long long) { return lift(v); }
    __device__ static A comb(A a, A b) { return __fadd_rn(a, b); }
    __device__ static A shfl(A a, int src) { return __shfl_sync(kFull, a, src); }
    __device__ static A shfl_up(A a, int d) { return __shfl_up_sync(kFull, a, d); }
    __device__ static A shfl_xor(A a, int m) { return __shfl_xor_sync(kFull, a, m); }
    __device__ static void store(void *o0, void *, uint64_t i, A a) { ((A *)o0)[i] = a; }
    __device__ static A load(const void *o0, const void *, uint64_t i) { return ((const A *)o0)[i]; }
    static constexpr int bytes0 = 4, bytes1 = 0;
};

template <>
struct AggT<22> {  // RS_OP_COUNT_MIN_U32 over uint32 elements: (count, min)
    static constexpr bool heavy = false;   // lift costs far more than a select (fused paths lift survivors only)
    static constexpr bool group = false;   // min has no inverse
    using A = uint2;
    __device__ static A id() { return make_uint2(0u, 0xffffffffu); }
    __device__ static A lift(uint32_t v) { return make_uint2(1u, v); }
    __device__ static A lift_i(uint32_t v, long long) { return lift(v); }
    __device__ static A comb(A a, A b) { return make_uint2(a.x + b.x, min(a.y, b.y)); }
    __device__ static A shfl(A a, int src) {
        return make_uint2(__shfl_sync(kFull, a.x, src), __shfl_sync(kFull, a.y, src));
    }
    __device__ static A shfl_up(A a, int d) {
        return make_uint2(__shfl_up_sync(kFull, a.x, d), __shfl_up_sync(kFull, a.y, d));
    }
    __device__ static A shfl_xor(A a, int m) {
        return make_uint2(__shfl_xor_sync(kFull, a.x, m), __shfl_xor_sync(kFull, a.y, m));
    }
    __device__ static void store(void *o0, void *o1, uint64_t i, A a) {
        ((uint32_t *)o0)[i] = a.x;
        ((uint32_t *)o1)[i] = a.y;
    }
    __device__ static A load(const void *o0, const void *o1, uint64_t i) {
        return make_uint2(((const uint32_t *)o0)[i], ((const uint32_t *)o1)[i]);
    }
    static constexpr int bytes0 = 4, bytes1 = 4;
};

// splitmix64 finalizer (reading A19: the text aggregate hashes (i << 8 | byte)).
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <>
struct AggT<23> {  // RS_OP_COUNT_XOR64 over u8 elements: (count, xor of mix64(i << 8 | byte))
    static constexpr bool heavy = true;   // lift costs far more than a select (fused paths lift survivors only)
    static constexpr bool group = true;   // count and xor both have exact inverses
    __device__ static ulonglong2 sub(ulonglong2 a, ulonglong2 b) { return make_ulonglong2(a.x - b.x, a.y ^ b.y); }
    using A = ulonglong2;
    __device__ static A id() { return make_ulonglong2(0ull, 0ull); }
    // item = byte | (position mod C) << 8; delta = chunk base - region start, so the
    // byte's index within its region is i = delta + (item >> 8)
    __device__ static A lift_i(uint32_t v, long long delta) {
        const unsigned long long i = (unsigned long long)(delta + (long long)(v >> 8));
        return make_ulonglong2(1ull, mix64((i << 8) | (v & 0xffu)));
    }
    __device__ static A lift(uint32_t v) { return lift_i(v, 0); }   // (index-free form; unused)
    __device__ static A comb(A a, A b) { return make_ulonglong2(a.x + b.x, a.y ^ b.y); }
    __device__ static A shfl(A a, int src) {
        return make_ulonglong2(__shfl_sync(kFull, a.x, src), __shfl_sync(kFull, a.y, src));
    }
    __device__ static A shfl_up(A a, int d) {
        return make_ulonglong2(__shfl_up_sync(kFull, a.x, d), __shfl_up_sync(kFull, a.y, d));
    }
    __device__ static A shfl_xor(A a, int m) {
        return make_ulonglong2(__shfl_xor_sync(kFull, a.x, m), __shfl_xor_sync(kFull, a.y, m));
    }
    __device__ static void store(void *o0, void *o1, uint64_t i, A a) {
        ((unsigned long long *)o0)[i] = a.x;
        ((unsigned long long *)o1)[i] = a.y;
    }
    __device__ static A load(const void *o0, const void *o1, uint64_t i) {
        return make_ulonglong2(((const unsigned long long *)o0)[i], ((const unsigned long long *)o1)[i]);
    }
    static constexpr int bytes0 = 8, bytes1 = 8;
};

template <>
struct AggT<24> {  // RS_OP_EMIT_VALUE: element-wise exit -- no per-region fold (the EMIT node writes items)
    static constexpr bool heavy = false;
    static constexpr bool group = true;
    using A = uint32_t;
    __device__ static A id() { return 0u; }
    __device__ static A lift(uint32_t) { return 0u; }
    __device__ static A lift_i(uint32_t, long long) { return 0u; }
    __device__ static A comb(A, A) { return 0u; }
    __device__ static A sub(A, A) { return 0u; }
    __device__ static A shfl(A a, int) { return a; }
    __device__ static A shfl_up(A a, int) { return a; }
    __device__ static A shfl_xor(A a, int) { return a; }
    __device__ static void store(void *, void *, uint64_t, A) {}
    __device__ static A load(const void *, const void *, uint64_t) { return 0u; }
    static constexpr int bytes0 = 4, bytes1 = 0;
};

template <>
struct AggT<25> : AggT<24> {};

// Fan-out (SPLIT node with two leaf SUM_I64 aggregates): the pair of sums, for
// the split-region partial slots and the fixup (v0 = child A, v1 = child B).
template <>
struct AggT<26> {
    static constexpr bool heavy = false;
    static constexpr bool group = true;
    using A = ulonglong2;
    __device__ static A id() { return make_ulonglong2(0ull, 0ull); }
    __device__ static A lift(uint32_t) { return id(); }
    __device__ static A lift_i(uint32_t, long long) { return id(); }
    __device__ static A comb(A a, A b) { return make_ulonglong2(a.x + b.x, a.y + b.y); }
    __device__ static A sub(A a, A b) { return make_ulonglong2(a.x - b.x, a.y - b.y); }
    __device__ static A shfl(A a, int src) {
        return make_ulonglong2(__shfl_sync(kFull, a.x, src), __shfl_sync(kFull, a.y, src));
    }
    __device__ static A shfl_up(A a, int d) {
        return make_ulonglong2(__shfl_up_sync(kFull, a.x, d), __shfl_up_sync(kFull, a.y, d));
    }
    __device__ static A shfl_xor(A a, int m) {
        return make_ulonglong2(__shfl_xor_sync(kFull, a.x, m), __shfl_xor_sync(kFull, a.y, m));
    }
    __device__ static void store(void *o0, void *o1, uint64_t i, A a) {
        ((unsigned long long *)o0)[i] = a.x;
        ((unsigned long long *)o1)[i] = a.y;
    }
    __device__ static A load(const void *o0, const void *o1, uint64_t i) {
        return make_ulonglong2(((const unsigned long long *)o0)[i], ((const unsigned long long *)o1)[i]);
    }
    static constexpr int bytes0 = 8, bytes1 = 8;
};   // RS_OP_EMIT_PAIR: element-wise exit of parsed "{x,y}" pairs (u8)

// SUM_I64 plus a per-region count carried by a node-generated signal
// (RS_OP_SUM_I64_DROPS): x = the int64 sum of the survivors, y = the items the
// first stage dropped (added by lane 0 when the signal arrives).
template <>
struct AggT<27> : AggT<26> {
    __device__ static A lift(uint32_t v) { return make_ulonglong2((unsigned long long)(long long)(int)v, 0ull); }
    __device__ static A lift_i(uint32_t v, long long) { return lift(v); }
};

template <class AT>
__device__ __forceinline__ typename AT::A warp_reduce(typename AT::A a) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) a = AT::comb(a, AT::shfl_xor(a, m));
    return a;
}

}  // namespace rs
