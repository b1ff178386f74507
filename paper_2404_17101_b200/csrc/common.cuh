// common.cuh -- shared device helpers for the B200-native FAST-BCC library (sm_100a).
#pragma once
#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>

typedef uint32_t u32;
typedef uint64_t u64;
typedef int64_t i64;

#define PG_INV 0xFFFFFFFFu

namespace pg {

// ---------------------------------------------------------------------------
// counter-based generator hash (rules pinned in DESIGN.md "Generators")
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ u64 sm64(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ u64 draw(u64 seed, u64 ctr) { return sm64(sm64(seed) ^ ctr); }

// ---------------------------------------------------------------------------
// L2-coherent loads/stores.  Union-find parents are mutated by other SMs inside the
// same kernel; L1 is not coherent, so parent reads bypass it (ld.global.cg).
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 ldcg(const u32* p) { return __ldcg(p); }
// L2 evict_last access policy and a read-only load under it
__device__ __forceinline__ u64 policy_evict_last() {
    u64 pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// (no L1 allocation: random gathers have no L1 reuse, and the L1 lines they would take
// hold other warps' in-flight data; C5a tags 36.7 -> 36.2 ms)
__device__ __forceinline__ u32 ld_keep(const u32* p, u64 pol) {
    u32 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ u32 ld_keep_l1(const u32* p, u64 pol) {
    u32 r;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
// random read-only gather without L1 allocation
__device__ __forceinline__ u32 ld_na(const u32* p) {
    u32 r;
    asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
// the same with the smallest L2 fetch hint: an isolated 4-byte gather otherwise brings a
// whole 128-byte line from DRAM (section 4.3 of DESIGN.md)
__device__ __forceinline__ u32 ld_na64(const u32* p) {
    u32 r;
    asm("ld.global.nc.L1::no_allocate.L2::64B.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ void stcg(u32* p, u32 v) { __stcg(p, v); }

__device__ __forceinline__ u64 ld_volatile_u64(const u64* p) {
    u64 v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(u64* p, u64 v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---------------------------------------------------------------------------
// Union-find over u32 parent arrays: link-by-index (larger root under smaller root),
// path halving with benign racing stores.  parent[x] <= x always, so every chain is
// strictly decreasing and halving never creates a cycle.  Each successful CAS merges two
// distinct trees, so the edges that won a CAS form a spanning forest.
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 uf_find(u32* P, u32 x) {
    for (;;) {
        u32 p = ldcg(P + x);
        if (p == x) return x;
        u32 gp = ldcg(P + p);
        if (gp == p) return p;
        stcg(P + x, gp);
        x = gp;
    }
}

// link a-b; returns true if this call merged two trees
__device__ __forceinline__ bool uf_link(u32* P, u32 a, u32 b) {
    u32 ra = uf_find(P, a), rb = uf_find(P, b);
    while (ra != rb) {
        u32 hi = ra > rb ? ra : rb, lo = ra ^ rb ^ hi;
        u32 old = atomicCAS(P + hi, hi, lo);
        if (old == hi) return true;
        ra = uf_find(P, ra);
        rb = uf_find(P, rb);
    }
    return false;
}

// Where a hook is recorded: HAB[2 hi] = {a, b} (each vertex is hooked at most once, so
// HAB names a spanning forest).  When the edge leaves hi itself (a == hi: arc 2hi; b == hi:
// arc 2hi+1) that "own" arc is also made the first entry of hi's out-arc list (HEAD[hi],
// NEXT[arc] = end) right here -- nothing else touches hi's list before the forest stage --
// so the forest stage's list building only inserts the other arcs (fewer returning
// exchanges).  HEAD == nullptr records the edge only.
struct HookRec {
    uint2* HAB;
    u32* HEAD;
    u32* NEXT;
    __device__ __forceinline__ void operator()(u32 hi, u32 a, u32 b) const {
        HAB[2 * (size_t)hi] = make_uint2(a, b);
        if (HEAD && (a == hi || b == hi)) {
            const u32 own = 2 * hi + (a == hi ? 0u : 1u);
            NEXT[own] = PG_INV;
            HEAD[hi] = own;
        }
    }
};

// link a-b and record the graph edge that caused the merge at the hooked root
__device__ __forceinline__ void uf_link_hook(u32* P, u32 a, u32 b, const HookRec& rec) {
    u32 ra = uf_find(P, a), rb = uf_find(P, b);
    while (ra != rb) {
        u32 hi = ra > rb ? ra : rb, lo = ra ^ rb ^ hi;
        u32 old = atomicCAS(P + hi, hi, lo);
        if (old == hi) {
            rec(hi, a, b);
            return;
        }
        ra = uf_find(P, ra);
        rb = uf_find(P, rb);
    }
}

__host__ __device__ __forceinline__ i64 cdiv(i64 a, i64 b) { return (a + b - 1) / b; }

}  // namespace pg

#define PG_CUDA_TRY(expr)                                  \
    do {                                                   \
        cudaError_t _e = (expr);                           \
        if (_e != cudaSuccess) return PASGAL_ECUDA;        \
    } while (0)

#define PG_LAUNCH_CHECK() PG_CUDA_TRY(cudaGetLastError())
