// bcc.cu -- FAST-BCC on one B200 (sm_100a): the hot path behind pasgal_bcc().
//
// Reference contract: pasgal.oracles.bcc_hopcroft_tarjan (oracles.py:119-201) output, the
// BccLabels parallel-mode labelling rule (results.py:76-88) and the spec'd but absent
// parallel module `bcc`, with corrections verified against the oracle
// (DESIGN.md section 3):
//   * fence(p,v) iff first[p] <= low[v] && high[v] <= last[p]   (SPEC.md:440 tests the
//     child's own interval, which is wrong);
//   * skeleton = non-fence tree edges + cross edges (back edges dropped);
//   * a non-root p is an articulation point iff some fence child c has comp[c] != comp[p]
//     (a fence child can share p's skeleton component through a cross edge).
//
// Stages (kernels), all stream-ordered, no host synchronisation:
//   S2 First-CC   k_cc_local (shared-memory union-find per id block; chunk row partition),
//                 k_cc_sample, k_compress, k_giant, k_cc_rest(+heavy)
//                 union-find; the edge that wins each hook CAS is recorded (HAB) = forest
//   S3 rooting    k_arc_link, k_arc_close (root chain, isolated slots), ruling-set list ranking (k_lr_walk1,
//                 k_wyllie, k_lr_walk2), preorder scan (first/last/parent)   Euler tour
//   S4 tags       k_tags_blk (per slot, blocked chunks), k_rmq_block/level/query (sparse table)
//   S5 Last-CC    k_cc2_local (non-fence tree edges and high-tag cross edges inside preorder
//                 blocks, shared memory), k_cc2_links (the block-crossing ones), k_giant,
//                 k_cc2_rest(+heavy)
//   S6 labels     k_compress_final, k_artic, k_labels, k_finish
//   canonical     k_canon_count, scan, k_canon_min, k_canon_apply     (flag CANONICAL)
#include <cstdio>
#include <cstdlib>
#include <cub/block/block_reduce.cuh>
#include <nvtx3/nvToolsExt.h>
#include "common.cuh"
#include "scan.cuh"
#include "wchunk.cuh"
#include "../../include/pasgal_bcc.h"

namespace pg {

constexpr u32 VFLAG = 0x80000000u;     // tour payload: arc is a root's virtual down arc
// HAB[2x+1].x tags of trimmed edges.  Tour arcs hold positions there, which stay below the
// tags (n < 2^31 - 2).
constexpr u32 TAG_TRIM_A = 0xFFFFFFFEu; // edge x trimmed: its endpoint .x is a forest leaf
constexpr u32 TAG_TRIM_B = 0xFFFFFFFDu; // edge x trimmed: its endpoint .y is a forest leaf
#ifndef PG_LABELS_MINB
#define PG_LABELS_MINB 8
#endif
#ifndef PG_NSAMPLE
#define PG_NSAMPLE 2
#endif
#ifndef PG_LOCAL_LB
#define PG_LOCAL_LB 13
#endif
constexpr int NSAMPLE = PG_NSAMPLE;    // neighbours linked per vertex before giant detection
// List-ranking ruler spacing 2^lr_shift(n): long walks amortise the pointer jumping on big
// tours, but a walk is a chain of dependent loads, so small graphs (L2-resident, launch-
// and latency-bound) use short ones.  PASGAL_BCC_LR_SHIFT overrides it (sweeps).
static inline int lr_shift(i64 n) {
    const char* e = getenv("PASGAL_BCC_LR_SHIFT");
    const int v = e ? atoi(e) : 0;
    if (v >= 1 && v <= 10) return v;
    // measured (profiles/r01_sweeps.txt): C1 2^16 -> 3, C2 2^20 and C3 2^24 -> 4,
    // C4 2^25 -> 5-6, C5a 2^28 -> 6-7
    if (n < ((i64)1 << 18)) return 3;
    if (n < ((i64)1 << 25)) return 4;
    return n < ((i64)1 << 28) ? 6 : 7;
}
constexpr int GIANT_SAMPLES = 1024;
constexpr int HEAVY_GRID = 148 * 4;

struct Ctr {
    u32 r1;       // non-isolated roots (trees with >= 1 forest edge)
    u32 niso;     // isolated vertices (no forest arc): preorder slots [0, niso)
    u32 roothead; // 1 + down arc of the first root on the tour chain (0: empty; memset-safe)
    u32 giant;    // sampled largest component (First-CC)
    u32 giant2;   // sampled largest skeleton component (Last-CC)
    u32 ncomp;    // skeleton components
    u32 verr;     // validation error bits
    u32 nheavy;   // heavy rows queued by k_cc_rest (HEAVY front)
    u32 nheavy2;  // heavy rows queued by k_cc2_rest (HEAVY front)
    u32 nvheavy;  // very heavy rows queued by k_cc_rest (HEAVY back, from index n-1 down)
    u32 nvheavy2; // very heavy rows queued by k_cc2_rest (HEAVY back)
    u32 gcid;     // component id (head preorder rank) of the sampled giant skeleton component
    u32 nfr;      // VGC First-CC: claimed vertices whose rows await the frontier pass (FR)
    u32 ntrim;    // forest leaves kept off the Euler tour (placed after the preorder scan)
    u32 nbigp;    // parents with more than LEAF_RUN leaves (their leaf slots: k_leaf_runs)
    u32 cc_vgc;   // First-CC path chosen by k_cc_policy: 1 = VGC local searches, 0 = sampled union-find
};

// Kernels of the two First-CC paths are all launched (a static launch sequence, capturable
// in a CUDA graph); the ones of the path k_cc_policy did not choose return at once.
__device__ __forceinline__ bool gated_off(const u32* gate, u32 want) { return gate && ldcg(gate) != want; }


// --------------------------------------------------------------------------
// workspace carve-up (identical for sizing and use)
// --------------------------------------------------------------------------
struct Ws {
    u32 *P, *HEAD;
    uint2* HAB;   // per vertex v: HAB[2v] = hook edge {a, b}; HAB[2v+1] = tour positions of arcs 2v, 2v+1
    u32* NEXT;
    u32 *SPLEN[2], *SPNEXT[2];
    u32* TA;      // arc at each tour position (walk2)
    u32* TP;      // parent (source vertex) of the arc at each tour position
    u64* T;       // (position of twin << 32) | target vertex [| VFLAG], per tour position
    uint2* FL;
    u32* FIRST;
    u32 *PV, *E, *PPAR;
    uint2 *W, *PM, *ST;
    u32* FPF;     // [position] parent's position | fence << 31 (PG_INV at roots)
    u32* C;       // Last-CC union-find over preorder positions
    u32* CIDV;    // per vertex: preorder rank of its skeleton component's head
    u32* TQ;      // two-level tags: code boundaries (1 KB), then the packed code table
    u32* GBIT;    // per vertex bit: CIDV[v] == gcid (33 MB at 2^28: L2-resident)
    u32 *ROOTMARK, *UCNT, *UOFF, *CANON, *HEAVY;
    u32* CROW;
    u64* SCAN;
    Ctr* ctr;
    i64 nb, lv, ns, nch;
    u32 lrs;      // list-ranking ruler spacing = 1 << lrs
};

static inline i64 rmq_levels(i64 nb) {
    i64 lv = 1;
    while (((i64)1 << lv) <= nb) ++lv;
    return lv;
}

// Ruler-array capacity: the default spacing coarsens as n grows (lr_shift), so a graph
// just below a threshold can need more rulers than one just above it.  Sizing for the
// largest count any n' <= n needs keeps pasgal_bcc_workspace_bytes non-decreasing in n, so
// a workspace sized for the largest graph of a batch fits every smaller one.
static inline i64 ruler_capacity(i64 n, i64 ns) {
    const i64 T[3] = {(i64)1 << 18, (i64)1 << 25, (i64)1 << 28};
    const int S[3] = {3, 4, 6};
    for (int k = 0; k < 3; ++k)
        if (n >= T[k]) {
            const i64 c = cdiv(2 * (T[k] - 1), (i64)1 << S[k]) + 1;
            if (c > ns) ns = c;
        }
    return ns;
}

static size_t carve(Ws& w, char* base, i64 n, i64 m) {
    size_t o = 0;
    auto take = [&](size_t bytes) -> char* {
        o = (o + 255) & ~(size_t)255;
        char* p = base ? base + o : nullptr;
        o += bytes;
        return p;
    };
    i64 nn = n > 0 ? n : 1;
    i64 L = 2 * nn;
    w.nb = cdiv(nn, 32);
    w.lv = rmq_levels(w.nb);
    w.lrs = (u32)lr_shift(n);
    w.ns = cdiv(L, (i64)1 << w.lrs) + 1;   // + the head ruler
    const i64 ns_cap = ruler_capacity(n, w.ns);
    w.nch = num_chunks(m);
    i64 scan_items = L > m ? L : m;
    w.P = (u32*)take(4 * nn);
    w.HAB = (uint2*)take(16 * nn);
    w.HEAD = (u32*)take(4 * nn);
    w.NEXT = (u32*)take(4 * L);
    for (int b = 0; b < 2; ++b) {
        w.SPLEN[b] = (u32*)take(4 * ns_cap);
        w.SPNEXT[b] = (u32*)take(4 * ns_cap);
    }
    w.TA = (u32*)take(4 * L);
    w.TP = (u32*)take(4 * L);
    w.T = (u64*)take(8 * L);
    w.FL = (uint2*)take(8 * nn);
    w.FIRST = (u32*)take(4 * nn);
    w.PV = (u32*)take(4 * nn);
    w.E = (u32*)take(4 * nn);
    w.PPAR = (u32*)take(4 * nn);
    w.W = (uint2*)take(8 * nn);
    w.PM = (uint2*)take(8 * nn);
    w.ST = (uint2*)take(8 * w.nb * w.lv);
    w.FPF = (u32*)take(4 * nn);
    w.C = (u32*)take(4 * nn);
    w.CIDV = (u32*)take(4 * nn);
    w.GBIT = (u32*)take(4 * w.nb);
    w.ROOTMARK = (u32*)take(4 * nn);
    w.UCNT = (u32*)take(4 * nn);
    w.UOFF = (u32*)take(4 * nn);
    w.CANON = (u32*)take(4 * nn);
    w.HEAVY = (u32*)take(4 * nn);
    w.CROW = (u32*)take(4 * (w.nch + 1));
    w.TQ = (u32*)take(1024 + 4 * cdiv(nn, 4));   // two-level tags: boundaries + code table (<= 1 byte per vertex)
    w.SCAN = (u64*)take(scan_status_bytes(scan_items > nn ? scan_items : nn));
    w.ctr = (Ctr*)take(sizeof(Ctr));
    return o + 256;
}

// --------------------------------------------------------------------------
// S2: First-CC (spanning forest by union-find with hook capture; Afforest-style
// neighbour sampling, then skip the sampled giant component)
// --------------------------------------------------------------------------

__global__ void k_canon_init(i64 n, u32* UCNT, i64 nlab, u32* CANON) {
    i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) UCNT[v] = 0;
    if (v < nlab) CANON[v] = PG_INV;
}

// Local phase (the paper's vertical granularity control recast for the GPU): a CTA owns a
// block of LOCAL_B consecutive ids and runs union-find on the block's internal sampled
// edges in shared memory, then publishes flat parents P[v] = block root.  Chains along the
// block (grid rows, preorder paths) collapse at shared-memory latency instead of walking
// global memory; only block-crossing edges reach the global union-find.
constexpr int LOCAL_LB = PG_LOCAL_LB;
constexpr int LOCAL_B = 1 << LOCAL_LB;
constexpr int LOCAL_T = 512;
// Block size 2^lb: LOCAL_B ids unless that leaves the GPU idle -- small graphs (C1: 8 CTAs
// of 8192 ids on 148 SMs) take smaller blocks so at least ~2 CTAs per SM run.
// PASGAL_BCC_LOCAL_LB overrides it (sweeps).
static inline int local_lb(i64 n) {
    const char* e = getenv("PASGAL_BCC_LOCAL_LB");
    const int v = e ? atoi(e) : 0;
    if (v >= 6 && v <= LOCAL_LB) return v;
    int lb = LOCAL_LB;
    while (lb > 9 && cdiv(n, (i64)1 << lb) < 2 * 148) --lb;
    return lb;
}

__device__ __forceinline__ u32 sfind(volatile u32* sp, u32 x) {
    for (;;) {
        u32 p = sp[x];
        if (p == x) return x;
        u32 gp = sp[p];
        if (gp == p) return p;
        sp[x] = gp;
        x = gp;
    }
}

// link local ids a-b; returns the hooked local root (or PG_INV if already joined)
__device__ __forceinline__ u32 slink(u32* sp, u32 a, u32 b) {
    u32 ra = sfind(sp, a), rb = sfind(sp, b);
    while (ra != rb) {
        u32 hi = ra > rb ? ra : rb, lo = ra ^ rb ^ hi;
        if (atomicCAS(sp + hi, hi, lo) == hi) return hi;
        ra = sfind(sp, ra);
        rb = sfind(sp, rb);
    }
    return PG_INV;
}

// It also initialises its block's hook records and out-arc heads (no separate init pass;
// P is published for every id below, and Last-CC's C by k_cc2_local).
// It also writes the warp-chunk row partition: CROW[c] = the nonempty row holding slot
// c * WCH, from the row's own offsets (no per-chunk binary search; a hub row writes the
// entries of all the chunks that start inside it).
__global__ void __launch_bounds__(LOCAL_T) k_cc_local(i64 n, int lb, const i64* __restrict__ off,
                                                      const int32_t* __restrict__ tgt, u32* P, uint2* HAB,
                                                      u32* HEAD, u32* NEXT, u32* CROW, const u32* gate) {
    __shared__ u32 sp[LOCAL_B];
    if (gated_off(gate, 0)) return;
    const i64 b0 = (i64)blockIdx.x << lb;
    const int cnt = (int)(n - b0 < (1 << lb) ? n - b0 : (1 << lb));
    for (int i = threadIdx.x; i < cnt; i += LOCAL_T) {
        sp[i] = (u32)i;
        reinterpret_cast<uint4*>(HAB)[b0 + i] = make_uint4(PG_INV, PG_INV, 0u, 0u);   // whole 16-byte record
        HEAD[b0 + i] = PG_INV;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += LOCAL_T) {
        i64 v = b0 + i, a = off[v], b = off[v + 1];
        if (CROW)
            for (i64 c = cdiv(a, WCH); c * WCH < b; ++c) CROW[c] = (u32)v;
        for (int k = 0; k < NSAMPLE && a + k < b; ++k) {
            i64 w = tgt[a + k];
            if ((w >> lb) != blockIdx.x) continue;
            u32 hi = slink(sp, (u32)i, (u32)(w - b0));
            if (hi != PG_INV) HookRec{HAB, NEXT ? HEAD : nullptr, NEXT}((u32)(b0 + hi), (u32)v, (u32)w);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += LOCAL_T) P[b0 + i] = (u32)b0 + sfind(sp, (u32)i);
}

// sampled edges that cross blocks (the local phase took the rest).  The roots of v and of
// its sampled neighbours are found in lockstep (independent pointer chains in flight
// together), then the links are made one CAS each with the roots already known; a failed
// CAS (another thread moved a root) falls back to the general uf_link_hook.  C5a First-CC
// 11.3 -> 10.9 ms.
template <int K>
__device__ __forceinline__ void uf_find_lockstep(u32* P, u32 (&x)[K]) {
    bool more = true;
    while (more) {
        more = false;
        u32 p[K], gp[K];
#pragma unroll
        for (int j = 0; j < K; ++j) p[j] = ldcg(P + x[j]);
#pragma unroll
        for (int j = 0; j < K; ++j) gp[j] = p[j] != x[j] ? ldcg(P + p[j]) : p[j];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if (p[j] == x[j]) continue;          // x[j] is a root
            if (gp[j] != p[j]) {                 // path halving, as uf_find
                stcg(P + x[j], gp[j]);
                more = true;
            }
            x[j] = gp[j];
        }
    }
}

__device__ __forceinline__ void cc_sample_one(i64 v, int lb, const i64* __restrict__ off,
                                              const int32_t* __restrict__ tgt, u32* P, const HookRec& rec);
__global__ void k_cc_sample(i64 n, int lb, const i64* __restrict__ off, const int32_t* __restrict__ tgt, u32* P,
                            HookRec rec, const u32* gate) {
    const i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n || gated_off(gate, 0)) return;
    cc_sample_one(v, lb, off, tgt, P, rec);
}

__device__ __forceinline__ void cc_sample_one(i64 v, int lb, const i64* __restrict__ off,
                                              const int32_t* __restrict__ tgt, u32* P, const HookRec& rec) {
    i64 a = off[v], b = off[v + 1];
    u32 t[NSAMPLE], x[NSAMPLE + 1];
    bool act[NSAMPLE], any = false;
    x[0] = (u32)v;
#pragma unroll
    for (int k = 0; k < NSAMPLE; ++k) {
        act[k] = a + k < b;
        t[k] = act[k] ? (u32)tgt[a + k] : (u32)v;
        act[k] = act[k] && (t[k] >> lb) != (u32)(v >> lb);
        x[k + 1] = act[k] ? t[k] : (u32)v;
        any |= act[k];
    }
    if (!any) return;
    uf_find_lockstep(P, x);
    u32 rv = x[0], hooked[NSAMPLE], under[NSAMPLE];
    int nh = 0;
    bool fallback = false;
#pragma unroll
    for (int k = 0; k < NSAMPLE; ++k) {
        if (!act[k]) continue;
        if (fallback) {
            uf_link_hook(P, (u32)v, t[k], rec);
            continue;
        }
        u32 rb = x[k + 1];
        for (int j = 0; j < nh; ++j)           // a root this thread hooked now hangs under `under`
            if (rb == hooked[j]) rb = under[j];
        if (rb == rv) continue;
        const u32 hi = rv > rb ? rv : rb, lo = rv ^ rb ^ hi;
        if (atomicCAS(P + hi, hi, lo) == hi) {
            rec(hi, (u32)v, t[k]);
            hooked[nh] = hi;
            under[nh] = lo;
            ++nh;
            rv = lo;
        } else {
            uf_link_hook(P, (u32)v, t[k], rec);
            fallback = true;
        }
    }
}

// Full compression.  A find is a chain of dependent loads, so each thread walks
// COMPRESS_ILP chains in lockstep (positions v, v+stride, ...) to keep several in flight.
// First-CC's forest (after sampling: shallow trees under the hubs) compresses best with 4
// chains per thread, Last-CC's (over preorder positions: longer chains) with 16 (sweep:
// C5a Last-CC 12.2 -> 11.4 ms; First-CC is slower above 4).
constexpr int COMPRESS_ILP = 4, COMPRESS_ILP2 = 16;

// Entries below `lo` are known self-roots and are neither read nor written (Last-CC: the
// preorder slots [0, niso) of the isolated vertices, 63 % of the positions at C5a).
template <int ILP>
__device__ __forceinline__ void compress_ilp(i64 n, u32* P, u32 (&root)[ILP], i64 (&idx)[ILP], i64 lo = 0) {
    const i64 stride = (i64)gridDim.x * blockDim.x;
    const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    u32 x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
        idx[j] = t + j * stride;
        x[j] = idx[j] < n ? (idx[j] < lo ? (u32)idx[j] : ldcg(P + idx[j])) : 0u;
    }
    bool more = true;
    while (more) {
        more = false;
        u32 px[ILP];
#pragma unroll
        for (int j = 0; j < ILP; ++j) px[j] = idx[j] < n && idx[j] >= lo ? ldcg(P + x[j]) : x[j];
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
            if (px[j] != x[j]) {
                x[j] = px[j];
                more = true;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
        root[j] = x[j];
        if (idx[j] < n && idx[j] >= lo) stcg(P + idx[j], x[j]);
    }
}

// 16 chains per thread took 140 registers (one 256-thread block per SM); capped at 128, two
// blocks fit without spills (C5a Last-CC -0.1..0.3 ms)
#ifndef PG_CMP_MINB
#define PG_CMP_MINB 2
#endif
template <int ILP>
__global__ void __launch_bounds__(256, ILP >= 16 ? PG_CMP_MINB : 1) k_compress(i64 n, u32* P, const u32* gate,
                                                                               const u32* lo = nullptr) {
    if (gated_off(gate, 0)) return;
    u32 root[ILP];
    i64 idx[ILP];
    compress_ilp<ILP>(n, P, root, idx, lo ? (i64)*lo : 0);
}

// most frequent root among GIANT_SAMPLES seeded samples (ties -> smaller root).  Counts in
// a shared-memory open-addressing table (one insert per thread) instead of every thread
// scanning all samples (O(S^2) shared loads: 24 us per call, a visible share at C1).
constexpr int GIANT_HASH = 2 * GIANT_SAMPLES;
__global__ void __launch_bounds__(GIANT_SAMPLES) k_giant(i64 n, const u32* P, u64 seed, u32* out, const u32* gate) {
    if (gated_off(gate, 0)) return;
    __shared__ u32 hk[GIANT_HASH], hc[GIANT_HASH];
    typedef cub::BlockReduce<u64, GIANT_SAMPLES> BR;
    __shared__ typename BR::TempStorage tmp;
    const int t = threadIdx.x;
    for (int k = t; k < GIANT_HASH; k += GIANT_SAMPLES) {
        hk[k] = PG_INV;
        hc[k] = 0;
    }
    const u32 v = (u32)(draw(seed ^ 0x5EEDB1CCull, (u64)t) % (u64)n);
    const u32 r = ldcg(P + v);
    __syncthreads();
    u32 h = (r * 0x9E3779B1u) >> (32 - 11);      // GIANT_HASH = 2^11 slots
    for (;;) {
        const u32 k = atomicCAS(hk + h, PG_INV, r);
        if (k == PG_INV || k == r) break;
        h = (h + 1) & (GIANT_HASH - 1);
    }
    atomicAdd(hc + h, 1u);
    __syncthreads();
    const u32 cnt = hc[h];
    const u64 key = ((u64)cnt << 32) | (u64)(PG_INV - r);
    const u64 best = BR(tmp).Reduce(key, cub::Max());
    if (t == 0) *out = PG_INV - (u32)(best & 0xFFFFFFFFu);
}

// Rows outside the sampled giant component: a thread per vertex skips giant rows with one
// read; rows longer than HEAVY_ROW slots go to a list served by a block per row, so a
// stray hub never serialises on one thread, and rows longer than VHEAVY_ROW to a second
// list whose rows are split over every block (one block per 2M-slot row took 4 ms).
// Repeats of the previous slot's target (parallel edges) are skipped in the long rows.
constexpr int HEAVY_ROW = 64;
constexpr i64 VHEAVY_ROW = 1 << 16;

__device__ __forceinline__ void queue_heavy(i64 n, i64 len, u32 u, u32* heavy, u32* nh, u32* nvh) {
    if (len > VHEAVY_ROW) heavy[n - 1 - atomicAdd(nvh, 1u)] = u;
    else heavy[atomicAdd(nh, 1u)] = u;
}

__global__ void k_cc_rest(i64 n, const i64* __restrict__ off, const int32_t* __restrict__ tgt, u32* P, HookRec HAB,
                          Ctr* ctr, u32* heavy, const u32* gate) {
    const i64 u = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n || gated_off(gate, 0)) return;
    i64 a = off[u] + NSAMPLE, b = off[u + 1];
    if (a >= b || ldcg(P + u) == ctr->giant) return;
    if (b - a > HEAVY_ROW) {
        queue_heavy(n, b - a, (u32)u, heavy, &ctr->nheavy, &ctr->nvheavy);
        return;
    }
    for (i64 s = a; s < b; ++s) uf_link_hook(P, (u32)u, (u32)tgt[s], HAB);
}

template <int SKIP>
__global__ void k_cc_rest_heavy(i64 n, const i64* __restrict__ off, const int32_t* __restrict__ tgt, u32* P,
                                HookRec HAB, const Ctr* ctr, const u32* __restrict__ heavy, const u32* gate, u32 want) {
    if (gated_off(gate, want)) return;
    const u32 nh = ctr->nheavy, nvh = ctr->nvheavy;
    for (u32 h = blockIdx.x; h < nh; h += gridDim.x) {
        u32 u = heavy[h];
        i64 a = off[u] + SKIP, b = off[u + 1];
        for (i64 s = a + threadIdx.x; s < b; s += blockDim.x) {
            const int32_t w = tgt[s];
            if (s > off[u] && tgt[s - 1] == w) continue;
            uf_link_hook(P, u, (u32)w, HAB);
        }
    }
    for (u32 h = 0; h < nvh; ++h) {
        u32 u = heavy[n - 1 - h];
        i64 a = off[u] + SKIP, b = off[u + 1];
        for (i64 s = a + (i64)blockIdx.x * blockDim.x + threadIdx.x; s < b; s += (i64)gridDim.x * blockDim.x) {
            const int32_t w = tgt[s];
            if (s > off[u] && tgt[s - 1] == w) continue;
            uf_link_hook(P, u, (u32)w, HAB);
        }
    }
}

// --------------------------------------------------------------------------
// S2, VGC form (north-star item 2; the paper's vertical granularity control, PAPER.md
// "Vertical Granularity Control", SPEC.md vgc-engine local_search): for sparse graphs
// (grids, kNN, roads: few slots per vertex, large diameter) the spanning forest is grown by
// per-warp multi-hop local searches instead of sampled union-find.
//
//   k_vgc_search  persistent warps; warp k scans its id range for unclaimed vertices and
//                 makes each a seed (CAS P[v]: INV -> v).  From a seed it runs a bounded
//                 BFS-order local search: its queue lives in shared memory, 32 queued
//                 vertices are expanded at once (one per lane), every neighbour still
//                 unclaimed is claimed for the seed (CAS P[w]: INV -> seed) with the edge
//                 that reached it as its forest edge (HAB[w]), and the search stops once
//                 tau vertices are processed -- so one search advances many hops and a
//                 large-diameter graph needs no per-level global rounds.  A neighbour
//                 claimed by ANOTHER search joins the two search trees in the union-find
//                 over seeds (uf_link_hook: the hook edge is the forest edge).  Queue
//                 overflow, the queue left when the search stops, and rows longer than
//                 VGC_HEAVY slots go to the frontier list FR (their rows are not yet read).
//   k_vgc_rest    every vertex is claimed by now; the FR rows link their neighbours' trees
//                 (thread per row; long rows to the block-per-row list of k_cc_rest_heavy).
//
// P[w] = seed for a claimed vertex and P[s] = s (or its hook) for a seed, so the roots are
// exactly the never-hooked seeds (P[x] == x) and every other vertex owns one forest edge in
// HAB, which is all the later stages use.  Claims build one tree per search; each hook
// joins two union-find trees through one edge, so the edges form a spanning forest.
// --------------------------------------------------------------------------
constexpr int VGC_WARPS = 4;          // warps per block
#ifndef PG_VGC_Q
#define PG_VGC_Q 256
#endif
constexpr int VGC_Q = PG_VGC_Q;            // per-warp queue capacity (ring of (vertex, seed), shared memory)
constexpr int VGC_HEAVY = 32;         // longer rows are deferred to the frontier pass
constexpr int VGC_TAU_DEFAULT = 1024; // vertices processed per local search (SPEC tau)

// First-CC policy, on the device (no host synchronisation): VGC local searches for a
// sparse graph (at most VGC_MAX_DEG slots per vertex on average) whose ids are LOCAL -- the
// first neighbour of most sampled vertices lies within n/256 ids (grids, meshes, road
// networks in their usual orderings) -- so that the searches' row reads and claims stay in
// cache; sampled union-find with the giant-component skip otherwise (dense or power-law
// graphs, where it reads only a few slots of most rows, and random-id graphs such as C4's
// kNN, where a search's every row read is a random line).  mode 1/2 forces VGC/union-find.
constexpr i64 VGC_MAX_DEG = 8;
constexpr i64 VGC_MIN_N = 1 << 18;   // below: launch/latency-bound, the id-block path is faster (C1)
constexpr int POLICY_SAMPLES = 1024;
__global__ void __launch_bounds__(POLICY_SAMPLES) k_cc_policy(i64 n, i64 m, const i64* __restrict__ off,
                                                              const int32_t* __restrict__ tgt, u64 seed, int mode,
                                                              Ctr* ctr) {
    __shared__ u32 nloc, nsamp;
    if (threadIdx.x == 0) nloc = nsamp = 0;
    __syncthreads();
    const u32 v = (u32)(draw(seed ^ 0x9011C7ull, threadIdx.x) % (u64)n);
    const i64 a = off[v], b = off[(i64)v + 1];
    if (b > a) {
        const i64 w = tgt[a];
        const i64 d = w > (i64)v ? w - (i64)v : (i64)v - w;
        atomicAdd(&nsamp, 1u);
        if (d <= (n >> 8) || d <= 64) atomicAdd(&nloc, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0)
        ctr->cc_vgc = mode == 1   ? 1u
                      : mode == 2 ? 0u
                                  : (n >= VGC_MIN_N && m <= VGC_MAX_DEG * n && 2 * nloc > nsamp) ? 1u : 0u;
}

__global__ void k_vgc_init(i64 n, const i64* __restrict__ off, u32* P, uint2* HAB, u32* HEAD, u32* CROW,
                           const u32* gate) {
    if (gated_off(gate, 1)) return;
    for (i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (i64)gridDim.x * blockDim.x) {
        P[v] = PG_INV;
        reinterpret_cast<uint4*>(HAB)[v] = make_uint4(PG_INV, PG_INV, 0u, 0u);
        HEAD[v] = PG_INV;
        if (CROW) {
            const i64 a = off[v], b = off[v + 1];
            for (i64 c = cdiv(a, WCH); c * WCH < b; ++c) CROW[c] = (u32)v;
        }
    }
}

__device__ __forceinline__ void vgc_push_frontier(u32* FR, Ctr* ctr, bool push, u32 x, int lane) {
    const unsigned pm = __ballot_sync(0xFFFFFFFFu, push);
    if (!pm) return;
    const int lead = __ffs(pm) - 1;
    u32 base = 0;
    if (lane == lead) base = atomicAdd(&ctr->nfr, (u32)__popc(pm));
    base = __shfl_sync(0xFFFFFFFFu, base, lead);
    if (push) FR[base + __popc(pm & ((1u << lane) - 1u))] = x;
}

// The warp's search loop.  Queue entries are (vertex, seed of its tree).  Each step
// expands up to 32 queued vertices at once: their rows are flattened over the lanes (a scan
// of the row lengths; each lane finds its slot's row by a 5-step shuffle search), and
// VGC_K slots per lane go through target load, claim check and claim CAS together, so a
// step costs a few dependent memory round trips whatever the row lengths.  Whenever fewer
// than 32 vertices are queued the warp starts new searches from the next unclaimed ids of
// its range, so the many small clusters of a sparse graph (a p = 0.6 grid) are searched
// several at a time instead of one short, latency-bound search after another.  After tau
// expansions the queue is flushed to the frontier and the warp starts afresh.
constexpr int VGC_K = 4;
__global__ void __launch_bounds__(VGC_WARPS * 32, 8) k_vgc_search(i64 n, const i64* __restrict__ off,
                                                               const int32_t* __restrict__ tgt, u32* P, HookRec HAB,
                                                               u32* FR, Ctr* ctr, int tau, const u32* gate) {
    __shared__ uint2 qs[VGC_WARPS][VGC_Q];
    if (gated_off(gate, 1)) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    uint2* Q = qs[wib];
    const i64 nw = (i64)gridDim.x * VGC_WARPS;
    const i64 wid = (i64)blockIdx.x * VGC_WARPS + wib;
    const i64 r0 = n * wid / nw, r1 = n * (wid + 1) / nw;
    i64 v0 = r0 - 32;          // current scan group [v0, v0 + 32)
    unsigned cm = 0;           // its unclaimed candidates not yet tried
    bool scanning = r0 < r1;
    u32 head = 0, tail = 0;    // monotone counters; slot = counter % VGC_Q
    int processed = 0;
    for (;;) {
        // refill with new seeds while the next step would run below a full warp
        while (scanning && tail - head < 32u) {
            if (!cm) {
                v0 += 32;
                if (v0 >= r1) {
                    scanning = false;
                    break;
                }
                const i64 v = v0 + lane;
                cm = __ballot_sync(0xFFFFFFFFu, v < r1 && ldcg(P + v) == PG_INV);
                continue;
            }
            const u32 need = 32u - (tail - head);
            unsigned take = cm;                         // the first `need` candidates
            while ((u32)__popc(take) > need) take &= ~(1u << (31 - __clz(take)));
            cm &= ~take;
            const u32 v = (u32)(v0 + lane);
            bool ok = false;
            if ((take >> lane) & 1u) ok = atomicCAS(P + v, PG_INV, v) == PG_INV;
            const unsigned okm = __ballot_sync(0xFFFFFFFFu, ok);
            if (ok) Q[(tail + (u32)__popc(okm & lt)) % VGC_Q] = make_uint2(v, v);
            tail += (u32)__popc(okm);
        }
        if (head == tail) break;
        const u32 cnt = tail - head < 32u ? tail - head : 32u;
        const bool has = (u32)lane < cnt;
        const uint2 ent = has ? Q[(head + lane) % VGC_Q] : make_uint2(0u, 0u);
        const u32 u = ent.x, sd = ent.y;
        head += cnt;
        processed += (int)cnt;
        i64 a = 0, b = 0;
        if (has) {
            a = off[u];
            b = off[(i64)u + 1];
        }
        const bool heavy = has && b - a > VGC_HEAVY;
        vgc_push_frontier(FR, ctr, heavy, u, lane);
        const u32 deg = has && !heavy ? (u32)(b - a) : 0u;
        u32 incl = deg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        const u32 total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        const u32 excl = incl - deg;
        u32 last_o = PG_INV;
        for (u32 base = 0; base < total; base += 32 * VGC_K) {
            u32 w[VGC_K], su[VGC_K], ss[VGC_K], o[VGC_K];
            bool act[VGC_K], claimed[VGC_K];
#pragma unroll
            for (int k = 0; k < VGC_K; ++k) {
                const u32 t = base + 32 * k + lane;
                act[k] = t < total;
                int j = 0;
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const u32 ex = __shfl_sync(0xFFFFFFFFu, excl, j + step < 32 ? j + step : 31);
                    if (j + step < 32 && ex <= t) j += step;
                }
                su[k] = __shfl_sync(0xFFFFFFFFu, u, j);
                ss[k] = __shfl_sync(0xFFFFFFFFu, sd, j);
                const i64 aj = __shfl_sync(0xFFFFFFFFu, a, j);
                const u32 ej = __shfl_sync(0xFFFFFFFFu, excl, j);
                w[k] = act[k] ? (u32)tgt[aj + (t - ej)] : 0u;
            }
#pragma unroll
            for (int k = 0; k < VGC_K; ++k) o[k] = act[k] ? ldcg(P + w[k]) : ss[k];
#pragma unroll
            for (int k = 0; k < VGC_K; ++k) {
                claimed[k] = false;
                if (o[k] == PG_INV) {
                    o[k] = atomicCAS(P + w[k], PG_INV, ss[k]);
                    if (o[k] == PG_INV) {
                        claimed[k] = true;
                        HAB(w[k], su[k], w[k]);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < VGC_K; ++k) {
                if (act[k] && !claimed[k] && o[k] != ss[k] && o[k] != last_o) {   // another tree: join
                    uf_link_hook(P, su[k], w[k], HAB);
                    last_o = o[k];
                }
                const unsigned cb = __ballot_sync(0xFFFFFFFFu, claimed[k]);
                if (cb) {
                    const u32 room = VGC_Q - (tail - head);
                    const u32 r = (u32)__popc(cb & lt);
                    const bool fits = claimed[k] && r < room;
                    if (fits) Q[(tail + r) % VGC_Q] = make_uint2(w[k], ss[k]);
                    vgc_push_frontier(FR, ctr, claimed[k] && !fits, w[k], lane);
                    const u32 tot = (u32)__popc(cb);
                    tail += tot < room ? tot : room;
                }
            }
        }
        __syncwarp();
        if (processed >= tau) {     // flush: the unexpanded queue's rows go to the frontier pass
            const u32 rem = tail - head;
            if (rem) {
                u32 fb = 0;
                if (lane == 0) fb = atomicAdd(&ctr->nfr, rem);
                fb = __shfl_sync(0xFFFFFFFFu, fb, 0);
                for (u32 q = lane; q < rem; q += 32) FR[fb + q] = Q[(head + q) % VGC_Q].x;
            }
            head = tail;
            processed = 0;
            __syncwarp();
        }
    }
}

// frontier rows: link every neighbour's tree (all vertices are claimed); long rows go to
// the block-per-row list (k_cc_rest_heavy with skip 0)
__global__ void k_vgc_rest(i64 n, const i64* __restrict__ off, const int32_t* __restrict__ tgt, u32* P, HookRec HAB,
                           const u32* __restrict__ FR, Ctr* ctr, u32* heavy, const u32* gate) {
    if (gated_off(gate, 1)) return;
    const u32 nfr = ctr->nfr;
    for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < nfr; k += gridDim.x * blockDim.x) {
        const u32 u = FR[k];
        const i64 a = off[u], b = off[(i64)u + 1];
        if (b - a > HEAVY_ROW) {
            queue_heavy(n, b - a, u, heavy, &ctr->nheavy, &ctr->nvheavy);
            continue;
        }
        const u32 ou = ldcg(P + u);
        for (i64 sl = a; sl < b; ++sl) {
            const u32 w = (u32)tgt[sl];
            if (ldcg(P + w) != ou) uf_link_hook(P, u, w, HAB);
        }
    }
}

// --------------------------------------------------------------------------
// S3: rooting by an Euler tour of the spanning forest.
//
// Arc space [0, 2n): a hooked vertex x owns the two arcs of its forest edge HAB[x]={a,b}:
// 2x = a->b and 2x+1 = b->a, so twin(arc) = arc^1.  A root r (never hooked) owns its two
// virtual arcs: 2r = down into r, 2r+1 = up out of r.  Around every vertex the out-arcs
// form a circular list NEXT (built with warp-aggregated atomicExch on HEAD[v]); the tour
// successor is then uniformly succ(arc) = NEXT[arc^1].  A root's cycle is cut at its up
// arc and the non-isolated roots are chained (in arbitrary order, by warp-aggregated
// atomicExch on a global head), so the forest is one list headed by that chain's head.  Isolated vertices (half of an RMAT graph) stay off
// the tour: the root scan gives them preorder slots [0, NISO) directly, and the tour's
// vertices take [NISO, n).
// --------------------------------------------------------------------------

// Insert arcs at the heads of their keys' circular out-arc lists.  Lanes naming the same
// key (hubs) are chained locally and spliced in with one atomicExch; each thread pushes
// its two arcs with both exchanges in flight before either result is used.
struct ArcGroup {
    unsigned grp;
    int lead;
    unsigned later;
};
__device__ __forceinline__ ArcGroup arc_group(u32 key, bool active, int lane) {
    ArcGroup g{0u, 0, 0u};
    unsigned act = __ballot_sync(0xFFFFFFFFu, active);
    if (active) {
        g.grp = __match_any_sync(act, key);
        g.lead = __ffs(g.grp) - 1;
        g.later = g.grp & (lane == 31 ? 0u : (0xFFFFFFFEu << lane));
    }
    return g;
}
__device__ __forceinline__ void arc_splice(u32* NEXT, const ArcGroup& g, u32 arc, u32 old) {
    old = __shfl_sync(g.grp, old, g.lead);
    u32 nxt = __shfl_sync(g.grp, arc, g.later ? __ffs(g.later) - 1 : (threadIdx.x & 31));
    NEXT[arc] = g.later ? nxt : old;   // the group's last arc continues into the old list
}

// Block-aggregated form (default): a block's AL_T hooked vertices insert their 2 AL_T arcs
// into a shared-memory table keyed by source vertex, chaining arcs of one source locally
// (shared-memory exchanges), then splice each local chain into the global list with ONE
// atomicExch per distinct source per block.  On a power-law forest most arcs leave a few
// hubs: per-warp aggregation still left ~5M returning exchanges on the top hub's HEAD,
// serialised at one L2 slice; per-block aggregation divides that by the block size and
// keeps each hub's list in runs of consecutive hooked ids.
#ifndef PG_AL_LOG
#define PG_AL_LOG 9
#endif
constexpr int AL_T = 1 << PG_AL_LOG, AL_H = 4 * AL_T;   // <= 2 keys per thread: the table stays half empty
// Leaf trimming: a non-root vertex of forest degree 1 is a leaf of the rooted forest
// whatever the rooting (C5a: most forest vertices are leaves hooked onto hubs), so its edge
// is kept off the Euler tour.  The edge's record gets a tag naming the leaf end and the
// leaf's rank among its parent's leaves; LCNT[p] counts p's leaves.  Ranks come from the
// same shared table (one global atomicAdd per parent per block).  The preorder scan then
// weighs every tour vertex by 1 + its leaf count, and k_vertex_first puts the leaves of p
// right after p.  fm.ONE == nullptr: no trimming.
//
// Forest marks (k_forest_marks): three n-bit maps, L2-resident (33 MB each at C5a):
// ONE = endpoint of >= 1 forest edge, TWO = of >= 2, ROOT = never hooked.
struct ForestMarks {
    u32 *ONE, *TWO, *ROOT;
    u32* LEAF;   // ONE & ~TWO & ~ROOT, written over TWO by k_leaf_bits
};
__device__ __forceinline__ bool fm_bit(const u32* bm, u32 v) { return (__ldcg(bm + (v >> 5)) >> (v & 31)) & 1u; }
__device__ __forceinline__ bool forest_leaf(u32 v, const ForestMarks& fm) { return fm_bit(fm.LEAF, v); }
__global__ void __launch_bounds__(AL_T) k_arc_link_blk(i64 n, uint2* HAB, u32* HEAD, u32* NEXT, bool own_placed,
                                                       ForestMarks fm, u32* LCNT, uint2* LPR, Ctr* ctr) {
    __shared__ u32 hkey[AL_H], hhead[AL_H], htail[AL_H], hleaf[AL_H];
    __shared__ u32 s_trim;
    for (int i = threadIdx.x; i < AL_H; i += AL_T) {
        hkey[i] = PG_INV;
        hhead[i] = PG_INV;
        hleaf[i] = 0;
    }
    if (threadIdx.x == 0) s_trim = 0;
    __syncthreads();
    const i64 x = (i64)blockIdx.x * AL_T + threadIdx.x;
    const uint2 e = x < n ? HAB[2 * x] : make_uint2(PG_INV, PG_INV);
    auto slot_of = [&](u32 key) -> u32 {
        u32 h = (key * 0x9E3779B1u) >> (32 - (PG_AL_LOG + 2));   // AL_H slots
        for (;;) {
            const u32 k = atomicCAS(hkey + h, PG_INV, key);
            if (k == PG_INV || k == key) return h;
            h = (h + 1) & (AL_H - 1);
        }
    };
    int lh = -1;                    // trimmed edge: the parent's slot
    u32 lrank = 0, ltag = 0;
    if (e.x != PG_INV) {
        const bool la = fm.ONE && forest_leaf(e.x, fm);
        const bool lb = fm.ONE && !la && forest_leaf(e.y, fm);
        if (la || lb) {
            lh = (int)slot_of(la ? e.y : e.x);
            lrank = atomicAdd(hleaf + lh, 1u);
            ltag = la ? TAG_TRIM_A : TAG_TRIM_B;
        } else {
#pragma unroll
            for (int d = 0; d < 2; ++d) {
                const u32 key = d ? e.y : e.x, arc = 2 * (u32)x + d;
                if (own_placed && key == (u32)x) continue;  // own arc: placed when x was hooked (HookRec)
                const u32 h = slot_of(key);
                const u32 old = atomicExch(hhead + h, arc);
                if (old == PG_INV) htail[h] = arc;             // first in: the local chain's tail
                else NEXT[arc] = old;
            }
        }
    }
    const unsigned tb = __ballot_sync(0xFFFFFFFFu, lh >= 0);
    if ((threadIdx.x & 31) == 0 && tb) atomicAdd(&s_trim, (u32)__popc(tb));
    __syncthreads();
    u32 key[AL_H / AL_T], old[AL_H / AL_T], lbase[AL_H / AL_T];
#pragma unroll
    for (int j = 0; j < AL_H / AL_T; ++j) {                 // the global atomics in flight together
        const int h = threadIdx.x + j * AL_T;
        key[j] = hkey[h];
        old[j] = key[j] != PG_INV && hhead[h] != PG_INV ? atomicExch(HEAD + key[j], hhead[h]) : 0u;
        lbase[j] = key[j] != PG_INV && hleaf[h] ? atomicAdd(LCNT + key[j], hleaf[h]) : 0u;
    }
#pragma unroll
    for (int j = 0; j < AL_H / AL_T; ++j) {
        const int h = threadIdx.x + j * AL_T;
        if (key[j] != PG_INV && hhead[h] != PG_INV) NEXT[htail[h]] = old[j];
        hleaf[h] = lbase[j];                                 // now: this block's first rank at the parent
    }
    if (threadIdx.x == 0 && s_trim) atomicAdd(&ctr->ntrim, s_trim);
    __syncthreads();
    // the whole 16-byte record (an 8-byte half would leave partially written sectors); the
    // leaf's (parent, rank) by vertex for k_vertex_first
    if (lh >= 0) {
        reinterpret_cast<uint4*>(HAB)[x] = make_uint4(e.x, e.y, ltag, hleaf[lh] + lrank);
        LPR[ltag == TAG_TRIM_A ? e.x : e.y] = make_uint2(ltag == TAG_TRIM_A ? e.y : e.x, hleaf[lh] + lrank);
    }
}

__global__ void k_leaf_bits(i64 nw, ForestMarks fm) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nw) fm.LEAF[i] = fm.ONE[i] & ~fm.TWO[i] & ~fm.ROOT[i];
}

// Forest marks (maps zeroed before): ROOT by one coalesced word per warp, ONE/TWO by
// warp-aggregated atomicOr on the endpoints of every hook edge (a second sighting sets TWO;
// lanes naming the same vertex count as sightings too)
__global__ void k_forest_marks(i64 n, const uint2* __restrict__ HAB, ForestMarks fm) {
    const i64 x = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const uint2 e = x < n ? HAB[2 * x] : make_uint2(0u, 0u);
    const bool hooked = x < n && e.x != PG_INV;
    const unsigned rb = __ballot_sync(0xFFFFFFFFu, x < n && !hooked);
    if (lane == 0 && x < n) fm.ROOT[x >> 5] = rb;
    const unsigned act = __ballot_sync(0xFFFFFFFFu, hooked);
    if (!hooked) return;
    // both endpoints' words read together (one L2 round trip), then at most one returning
    // atomic per endpoint group
    u32 v[2], t[2], o[2];
    bool lead[2], many[2];
#pragma unroll
    for (int d = 0; d < 2; ++d) {
        v[d] = d ? e.y : e.x;
        const unsigned grp = __match_any_sync(act, v[d]);
        lead[d] = lane == __ffs(grp) - 1;
        many[d] = __popc(grp) > 1;
    }
#pragma unroll
    for (int d = 0; d < 2; ++d) {
        t[d] = lead[d] ? __ldcg(fm.TWO + (v[d] >> 5)) : 0u;
        o[d] = lead[d] ? __ldcg(fm.ONE + (v[d] >> 5)) : 0u;
    }
#pragma unroll
    for (int d = 0; d < 2; ++d) {
        const u32 bit = 1u << (v[d] & 31);
        if (!lead[d] || (t[d] & bit)) continue;     // a hub's bits are set after its first sightings
        bool second = many[d] || (o[d] & bit);
        if (!(o[d] & bit)) {                         // ONE must hold for every endpoint (isolated test)
            const u32 old = atomicOr(fm.ONE + (v[d] >> 5), bit);
            second = second || (old & bit);
        }
        if (second) atomicOr(fm.TWO + (v[d] >> 5), bit);
    }
}


// Close every out-arc list into a cycle (a root's cycle exits through its up arc).  Roots:
//   isolated (no forest arc): preorder slot f from a warp-aggregated counter; only FL[v] is
//   written (no pass over positions reads the records of a slot below niso);
//   otherwise succ(2r) = NEXT[2r+1] = first out-arc of r, and succ(2r+1) = NEXT[2r] = the
//   down arc of the root chained before r (warp-aggregated atomicExch on ctr->roothead).
// Neither the order of trees on the tour nor the order of isolated slots matters.

struct IsoOut {
    uint2* FL;
    u32* ROOTMARK;
};

// One block = AC_B threads x AC_V vertices.  Both the isolated-slot counter and the root
// chain are aggregated in shared memory first, so each block issues at most three global
// atomics (a single global head hit once per warp serialised ~8M atomics at RMAT 2^28).
constexpr int AC_B = 512, AC_V = 8;

__global__ void __launch_bounds__(AC_B) k_arc_close(i64 n, uint2* HAB, const u32* __restrict__ HEAD,
                                                    const u32* __restrict__ P, ForestMarks fm,
                                                    Ctr* ctr, u32* NEXT, IsoOut io) {
    __shared__ u32 s_niso, s_r1, s_head, s_tail, s_base;
    if (threadIdx.x == 0) { s_niso = 0; s_r1 = 0; s_head = 0; s_tail = PG_INV; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const i64 base = (i64)blockIdx.x * (AC_B * AC_V) + threadIdx.x;
    u32 slot[AC_V];
#pragma unroll
    for (int i = 0; i < AC_V; ++i) {
        const i64 x = base + (i64)i * AC_B;
        const uint4 rec = x < n ? reinterpret_cast<const uint4*>(HAB)[x] : make_uint4(0u, 0u, 0u, 0u);
        const uint2 e = make_uint2(rec.x, rec.y);
        const bool root = x < n && e.x == PG_INV;
        const u32 h = root ? HEAD[x] : PG_INV;
        // isolated: no forest edge (with trimming a root whose children are all leaves has
        // an empty out-arc list but stays on the tour, down and straight back up)
        const bool iso = root && (fm.ONE ? !fm_bit(fm.ONE, (u32)x) : h == PG_INV);
        const bool chain = root && !iso;
        const bool trimmed = rec.z == TAG_TRIM_A || rec.z == TAG_TRIM_B;
        if (x < n && !root && !trimmed) {
#pragma unroll
            for (int d = 0; d < 2; ++d) {
                u32 arc = 2 * (u32)x + d;
                if (NEXT[arc] == PG_INV) {          // tail of the list of its source vertex
                    u32 src = d == 0 ? e.x : e.y;
                    NEXT[arc] = P[src] == src ? 2 * src + 1 : HEAD[src];
                }
            }
        }
        // isolated vertices: block-local slot, made global after the block's one atomicAdd
        const unsigned bi = __ballot_sync(0xFFFFFFFFu, iso);
        u32 lb = 0;
        if (bi && lane == __ffs(bi) - 1) lb = atomicAdd(&s_niso, (u32)__popc(bi));
        lb = __shfl_sync(0xFFFFFFFFu, lb, bi ? __ffs(bi) - 1 : 0);
        slot[i] = iso ? lb + (u32)__popc(bi & lt) : PG_INV;
        // non-isolated roots: the warp's roots form a local chain spliced into the block chain
        const unsigned bc = __ballot_sync(0xFFFFFFFFu, chain);
        if (bc) {
            const int lead = __ffs(bc) - 1;
            u32 old = 0;
            if (lane == lead) {
                old = atomicExch(&s_head, 2 * (u32)x + 1);
                atomicAdd(&s_r1, (u32)__popc(bc));
            }
            old = __shfl_sync(0xFFFFFFFFu, old, lead);
            const unsigned later = bc & (lane == 31 ? 0u : (0xFFFFFFFEu << lane));
            const u32 nxt = __shfl_sync(0xFFFFFFFFu, 2 * (u32)x, later ? __ffs(later) - 1 : lane);
            if (chain) {
                // down into r, then its first out-arc -- or, when all of r's children are
                // trimmed leaves, straight back up: succ(2r) = NEXT[2r+1] = 2r+1
                NEXT[2 * x + 1] = h != PG_INV ? h : 2 * (u32)x + 1;
                if (later) NEXT[2 * x] = nxt;         // up out of r, then the next root's down arc
                else if (old) NEXT[2 * x] = old - 1;
                else s_tail = 2 * (u32)x;             // block tail: linked to the global chain
                io.ROOTMARK[x] = PG_INV;              // root articulation marker (k_artic)
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_niso) s_base = atomicAdd(&ctr->niso, s_niso);
        if (s_head) {
            u32 old = atomicExch(&ctr->roothead, s_head);
            NEXT[s_tail] = old - 1;                   // 0 - 1 = PG_INV ends the tour
            atomicAdd(&ctr->r1, s_r1);
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < AC_V; ++i) {
        if (slot[i] == PG_INV) continue;
        const u32 v = (u32)(base + (i64)i * AC_B), f = s_base + slot[i];
        // nothing reads the per-position records (PV, E, PPAR, W) of an isolated slot: every
        // pass over positions starts at niso
        io.FL[v] = make_uint2(f, f);
    }
}

// ruling-set list ranking over succ(a) = NEXT[a^1].  Rulers: every on-tour arc a with
// a % 2^lrs == 0, plus the head (ruler index nsk).  walk1: each ruler's sublist length and
// next ruler; Wyllie on the rulers; walk2: final positions (into HAB[2y+1]) and TA[position] = arc.
struct TourInfo {
    u32 head;     // first arc of the list, PG_INV if the tour is empty
    u32 len;      // arcs on the tour = 2 * (n - isolated - trimmed leaves)
};
__device__ __forceinline__ TourInfo tour_info(const Ctr* ctr, i64 n) {
    TourInfo t;
    t.head = ctr->roothead - 1;                // PG_INV when no root is chained
    t.len = (u32)(2 * (n - (i64)ctr->niso - (i64)ctr->ntrim));
    return t;
}
// a ruler is an on-tour arc: not an arc of a trimmed leaf edge (record tag) nor of an
// isolated vertex (a root without forest edges: ONE map with trimming, empty list without)
__device__ __forceinline__ bool ruler_start(i64 s, i64 nsk, const TourInfo& t, const uint2* HAB, const u32* HEAD,
                                            const u32* ONE, u32 lrs, u32& x) {
    if (s < nsk) {
        x = (u32)s << lrs;
        const u32 v = x >> 1;
        const uint4 rec = reinterpret_cast<const uint4*>(HAB)[v];
        if (rec.z == TAG_TRIM_A || rec.z == TAG_TRIM_B) return false;
        if (rec.x != PG_INV) return true;
        return ONE ? ((ONE[v >> 5] >> (v & 31)) & 1u) != 0 : HEAD[v] != PG_INV;
    }
    x = t.head;
    return t.head != PG_INV && (t.head & ((1u << lrs) - 1u)) != 0;
}

__global__ void k_lr_walk1(i64 n, i64 ns, u32 lrs, const u32* __restrict__ NEXT, const uint2* __restrict__ HAB,
                           const u32* __restrict__ HEAD, const u32* __restrict__ ONE, const Ctr* ctr, u32* SPLEN,
                           u32* SPNEXT) {
    i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ns) return;
    const TourInfo t = tour_info(ctr, n);
    const i64 nsk = ns - 1;
    u32 x;
    if (!ruler_start(s, nsk, t, HAB, HEAD, ONE, lrs, x)) {
        SPLEN[s] = 0;
        SPNEXT[s] = PG_INV;
        return;
    }
    u32 cnt = 0;
    do {
        ++cnt;
        x = __ldg(NEXT + (x ^ 1u));
    } while (x != PG_INV && (x & ((1u << lrs) - 1u)) != 0);   // the head is never revisited
    SPLEN[s] = cnt;
    SPNEXT[s] = x == PG_INV ? PG_INV : x >> lrs;
}

// Wyllie pointer jumping on the rulers: suffix sums of sublist lengths
__global__ void k_wyllie(i64 ns, const u32* __restrict__ len_in, const u32* __restrict__ nxt_in, u32* len_out,
                         u32* nxt_out) {
    i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ns) return;
    u32 nx = nxt_in[s];
    u32 l = len_in[s];
    if (nx != PG_INV) {
        l += len_in[nx];
        nx = nxt_in[nx];
    }
    len_out[s] = l;
    nxt_out[s] = nx;
}

// All Wyllie rounds in one CTA when the rulers fit in shared memory (small graphs: C1 has
// 16K rulers and took 15 launches): SPLEN/SPNEXT[0] in, SPLEN[1] out.
constexpr int WY_T = 1024, WY_IPT = 20, WY_MAX = WY_T * WY_IPT;
__global__ void __launch_bounds__(WY_T) k_wyllie_small(i64 ns, const u32* __restrict__ len_in,
                                                       const u32* __restrict__ nxt_in, u32* len_out) {
    extern __shared__ u32 wy[];
    u32* L = wy;
    u32* X = wy + WY_MAX;
    for (i64 s = threadIdx.x; s < ns; s += WY_T) {
        L[s] = len_in[s];
        X[s] = nxt_in[s];
    }
    __syncthreads();
    for (;;) {
        u32 l[WY_IPT], x[WY_IPT];
        int live = 0;
#pragma unroll
        for (int j = 0; j < WY_IPT; ++j) {
            const i64 s = threadIdx.x + (i64)j * WY_T;
            if (s < ns) {
                l[j] = L[s];
                x[j] = X[s];
                if (x[j] != PG_INV) {
                    l[j] += L[x[j]];
                    x[j] = X[x[j]];
                    live |= x[j] != PG_INV;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < WY_IPT; ++j) {
            const i64 s = threadIdx.x + (i64)j * WY_T;
            if (s < ns) {
                L[s] = l[j];
                X[s] = x[j];
            }
        }
        if (!__syncthreads_or(live)) break;
    }
    for (i64 s = threadIdx.x; s < ns; s += WY_T) len_out[s] = L[s];
}

constexpr int LR_T = 256;

__global__ void __launch_bounds__(LR_T) k_lr_walk2(i64 n, i64 ns, u32 lrs, const u32* __restrict__ NEXT,
                                                   const uint2* __restrict__ HAB, const u32* __restrict__ HEAD,
                                                   const u32* __restrict__ ONE, const Ctr* ctr,
                                                   const u32* __restrict__ SUFFIX, uint2* HABW, u32* TA) {
    __shared__ __align__(16) u32 lr_buf[LR_T * 8];
    i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ns) return;
    const TourInfo t = tour_info(ctr, n);
    u32 x;
    if (!ruler_start(s, ns - 1, t, HAB, HEAD, ONE, lrs, x)) return;
    const u32 pos0 = t.len - SUFFIX[s];
    u32 pos = pos0;
    // TA[pos] = arc, staged per thread so that whole 32-byte sectors (8 positions, aligned)
    // are written at once: with ~8M walkers in flight a sector written 4 bytes at a time
    // leaves L2 half-filled and costs a read-modify-write in HBM
    u32* buf = lr_buf + threadIdx.x * 8;
    do {
        u32 nx = __ldg(NEXT + (x ^ 1u));   // issue the chain load first
        reinterpret_cast<u32*>(HABW + 2 * (i64)(x >> 1) + 1)[x & 1u] = pos;   // position of arc x
        buf[pos & 7u] = x;
        if ((pos & 7u) == 7u) {
            if (pos - 7u >= pos0) {
                const uint4* b4 = reinterpret_cast<const uint4*>(buf);
                uint4* d = reinterpret_cast<uint4*>(TA + (pos - 7u));
                d[0] = b4[0];
                d[1] = b4[1];
            } else {
                for (u32 q = pos0; q <= pos; ++q) TA[q] = buf[q & 7u];   // this walker's head sector
            }
        }
        ++pos;
        x = nx;
    } while (x != PG_INV && (x & ((1u << lrs) - 1u)) != 0);
    // the unfinished last sector (possibly also the first): positions [max(pos & ~7, pos0), pos)
    for (u32 q = (pos & ~7u) > pos0 ? (pos & ~7u) : pos0; q < pos; ++q) TA[q] = buf[q & 7u];
}

// preorder pass over tour positions, fused into a decoupled-look-back scan of the
// "down arc" flags (an arc is down iff it precedes its twin).  The load resolves the
// twin's position, the arc's target and its source (the parent, for a down arc) and
// stashes them in this tile's own T[k] / TA[k]: the store must not read another tile's
// items, which the look-back does not order.
struct PreLoad {
    const u32* TA;
    const uint2* HAB;
    u64* T;
    u32* TP;
    const Ctr* ctr;
    i64 n;
    const u32* LCNT;   // non-null with leaf trimming: a down arc weighs 1 + its vertex's leaves
    // all reads are read-only for the kernel (__ldg), so the compiler may issue the next
    // items' gathers before this item's stores
    __device__ __forceinline__ u32 operator()(i64 k) const {
        if (k >= (i64)tour_info(ctr, n).len) return 0u;
        u32 x = __ldg(TA + k);
        // one 16-byte record: the hook edge and both arcs' positions
        uint4 r = __ldg(reinterpret_cast<const uint4*>(HAB + 2 * (i64)(x >> 1)));
        u32 pt = (x & 1u) ? r.z : r.w;   // the twin's position
        uint2 e = make_uint2(r.x, r.y);
        u32 tg, src;
        if (e.x != PG_INV) {                 // tree arc 2y = a->b, 2y+1 = b->a
            tg = (x & 1u) ? e.x : e.y;
            src = (x & 1u) ? e.y : e.x;
        } else {                             // virtual arc of root y: parent = self
            tg = (x >> 1) | ((x & 1u) ? 0u : VFLAG);
            src = x >> 1;
        }
        T[k] = ((u64)pt << 32) | tg;
        TP[k] = src;
        if ((u64)k >= pt) return 0u;
        return LCNT ? 1u + __ldg(LCNT + (tg & ~VFLAG)) : 1u;
    }
};
struct PreStore {
    const u64* T;
    const u32* TP;
    const Ctr* ctr;
    uint2* FL;
    u32 *PV, *E, *PPAR;
    uint2* W;
    u32* PWX;          // non-null with leaf trimming: the weighted exclusive prefix per position
    i64 n;
    __device__ __forceinline__ void operator()(i64 k, u32 f, u32 down) const {
        if (PWX) {     // the per-vertex writes need the prefix at the twin: k_pre_place
            if (k < (i64)tour_info(ctr, n).len) PWX[k] = f;
            return;
        }
        if (!down) return;
        f += ctr->niso;                   // isolated vertices occupy [0, niso)
        u64 t = T[k];
        u32 pt = (u32)(t >> 32), lo = (u32)t;
        u32 v = lo & ~VFLAG;
        u32 last = f + (pt - (u32)k + 1) / 2 - 1;
        u32 par = TP[k];                 // source of the down arc p->v
        (void)lo;
        FL[v] = make_uint2(f, last);   // FIRST and the optional outputs: k_vertex_first
        PV[f] = v;
        E[f] = last;
        PPAR[f] = par;
        W[f] = make_uint2(f, f);
    }
};

// With leaf trimming: first = niso + the weighted prefix at the down arc, last = niso + the
// prefix at its twin (up) arc - 1 (the subtree's tour vertices and their leaves lie between)
// The slots of v's leaves follow v's own, so v also writes their E / PPAR / W (position
// order, coalesced); v's with more than LEAF_RUN leaves go to k_leaf_runs (a block each).
constexpr u32 LEAF_RUN = 32;
__global__ void k_pre_place(i64 n, const u64* __restrict__ T, const u32* __restrict__ TP,
                            const u32* __restrict__ PWX, Ctr* ctr, const u32* __restrict__ LCNT, uint2* FL, u32* PV,
                            u32* E, u32* PPAR, uint2* W, u32* bigp) {
    const i64 k = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (i64)tour_info(ctr, n).len) return;
    const u64 t = T[k];
    const u32 pt = (u32)(t >> 32);
    if ((u64)k >= pt) return;                   // up arc
    const u32 niso = ctr->niso;
    const u32 v = (u32)t & ~VFLAG;
    const u32 f = niso + PWX[k], last = niso + __ldg(PWX + pt) - 1u;
    FL[v] = make_uint2(f, last);
    PV[f] = v;
    E[f] = last;
    PPAR[f] = TP[k];
    W[f] = make_uint2(f, f);
    const u32 c = __ldg(LCNT + v);
    if (c > LEAF_RUN) {
        bigp[atomicAdd(&ctr->nbigp, 1u)] = v;
        return;
    }
    for (u32 r = 1; r <= c; ++r) {
        E[f + r] = f + r;
        PPAR[f + r] = v;
        W[f + r] = make_uint2(f + r, f + r);
    }
}

// leaf slots of the parents with many leaves: one block per parent, coalesced
__global__ void k_leaf_runs(const Ctr* ctr, const u32* __restrict__ bigp, const u32* __restrict__ LCNT,
                            const uint2* __restrict__ FL, u32* E, u32* PPAR, uint2* W) {
    const u32 nb = ctr->nbigp;
    for (u32 b = blockIdx.x; b < nb; b += gridDim.x) {
        const u32 v = bigp[b], c = LCNT[v], f = FL[v].x;
        for (u32 r = 1 + threadIdx.x; r <= c; r += blockDim.x) {
            E[f + r] = f + r;
            PPAR[f + r] = v;
            W[f + r] = make_uint2(f + r, f + r);
        }
    }
}


// FIRST[v] = FL[v].x and the optional parent/first outputs, per vertex and coalesced: the
// preorder store writes only FL by vertex (a random 8-byte write; a second random 4-byte
// FIRST write cost a partial-sector read-modify-write per vertex)
// With leaf trimming it also places the leaves (LEAF map): leaf v of parent p with rank r
// takes slot first[p] + 1 + r (E / PPAR / W of the slot were written by the parent).
__global__ void k_vertex_first(i64 n, uint2* FL, const u32* __restrict__ PPAR, u32* FIRST, u32* out_parent,
                               u32* out_first, const u32* __restrict__ LEAF, const uint2* __restrict__ LPR, u32* PV,
                               const Ctr* ctr) {
    const i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    u32 f;
    if (LEAF && ((LEAF[v >> 5] >> (v & 31)) & 1u)) {
        const uint2 pr = LPR[v];
        f = FL[pr.x].x + 1u + pr.y;
        FL[v] = make_uint2(f, f);
        PV[f] = (u32)v;
    } else {
        f = FL[v].x;
    }
    FIRST[v] = f;
    if (out_first) out_first[v] = f;
    if (out_parent) out_parent[v] = f < ctr->niso ? (u32)v : __ldg(PPAR + f);   // isolated: its own parent
}

// --------------------------------------------------------------------------
// S4: tags  w1/w2[first[v]] = min/max(first[v], first[u] for all neighbours u)
// --------------------------------------------------------------------------
__device__ __forceinline__ void write_tag(uint2* W, u32 f, u32 mn, u32 mx, bool atomic) {
    if (atomic) {
        atomicMin(&W[f].x, mn);
        atomicMax(&W[f].y, mx);
    } else {
        W[f] = make_uint2(mn < f ? mn : f, mx > f ? mx : f);
    }
}

// Blocked-chunk k_tags (wchunk.cuh): lane l reduces its 8 consecutive slots sequentially;
// a row wholly inside the lane is stored at once, and rows crossing lanes are combined by
// one segmented warp scan.  Rows that began before the chunk or continue after it use
// atomics.  The FIRST gathers themselves run in the strided layout (one instruction covers
// 32 consecutive slots: the sorted hub rows' targets share lines) and are transposed
// through shared memory.  It replaced a per-32-slot-window design (row search, segment
// mask, two redux and a carry per window) that was instruction-bound: C3 tags 0.50 ->
// 0.21 ms; C5a is gather-bound and unchanged (36.7 ms).
#ifndef PG_TAGS_MINB
#define PG_TAGS_MINB 6
#endif
// NOL1: the FIRST gathers skip L1 (large graphs: no reuse, and L1 holds in-flight misses);
// below 2^22 vertices FIRST (<= 16 MB) partly lives in L1 and the plain load is faster
template <bool NOL1>
__global__ void __launch_bounds__(WCH_BLOCK, PG_TAGS_MINB) k_tags_blk(const i64* __restrict__ off,
                                                                const int32_t* __restrict__ tgt, i64 n, i64 m,
                                                                const u32* __restrict__ crow,
                                                                const u32* __restrict__ FIRST, uint2* W,
                                                                u32* __restrict__ DIR) {
    __shared__ BlkSmem smem[WCH_BLOCK / 32];
    const int lane = threadIdx.x & 31;
    const i64 c = ((i64)blockIdx.x * WCH_BLOCK + threadIdx.x) >> 5;
    if (c >= num_chunks(m)) return;
    BlkSmem& sm = smem[threadIdx.x >> 5];
    const i64 s0 = c * WCH, s1 = s0 + WCH < m ? s0 + WCH : m;
    const i64 sl = s0 + BLK_SPL * lane;
    const u32 base = crow[c];
    // one row over the whole chunk (hub rows: most slots of a power-law graph): a plain
    // warp min/max, no row pass, no transpose, no scan
    const i64 a_base = off[base], e_base = off[(i64)base + 1];
    const bool one_row = e_base >= s1;
    u32 fw[BLK_SPL];
    {
        // FIRST lines are kept in L2 ahead of the W stores and offsets (evict_last): C5a
        // tags 36.8 -> 36.3 ms
        const u64 pol = policy_evict_last();
        u32 g[WCH_U];   // strided: one gather instruction covers 32 consecutive slots
        wc_load(tgt, m, c, lane, g);
#pragma unroll
        for (int k = 0; k < WCH_U; ++k)
            if (s0 + 32 * k + lane < s1) g[k] = NOL1 ? ld_keep(FIRST + g[k], pol) : ld_keep_l1(FIRST + g[k], pol);
        if (one_row) {   // warp-uniform
            const u32 fb = __ldg(FIRST + base);
            u32 mn = PG_INV, mx = 0, dw = 0;
#pragma unroll
            for (int k = 0; k < WCH_U; ++k) {
                const bool ok = s0 + 32 * k + lane < s1;
                if (ok) {
                    mn = g[k] < mn ? g[k] : mn;
                    mx = g[k] > mx ? g[k] : mx;
                }
                const unsigned b = __ballot_sync(0xFFFFFFFFu, ok && g[k] > fb);
                if (lane == k) dw = b;
            }
            if (DIR && lane < WCH_U) DIR[(i64)WCH_U * c + lane] = dw;
            mn = __reduce_min_sync(0xFFFFFFFFu, mn);
            mx = __reduce_max_sync(0xFFFFFFFFu, mx);
            if (lane == 0) write_tag(W, fb, mn, mx, a_base < s0 || e_base > s1);
            return;
        }
        blk_transpose(sm, lane, g, fw);
    }
    const BlkRows br = blk_rows(off, n, s0, s1, base, lane, sm);
    const bool hstart = br.mb & 1u;
    const u32 fh = __ldg(FIRST + br.r_first);    // the head row's preorder position
    u32 fr = fh;                                  // the current row's
    u32 mn = PG_INV, mx = 0, hmn = PG_INV, hmx = 0, db = 0;
    bool in_head = true;
#pragma unroll
    for (int i = 0; i < BLK_SPL; ++i) {
        if (i > 0 && (br.mb >> i & 1u)) {        // a row starts at slot i: the current one ended
            if (in_head) {
                hmn = mn;
                hmx = mx;
                in_head = false;
                if (hstart) write_tag(W, fr, mn, mx, false);   // began at p0: complete
            } else {
                write_tag(W, fr, mn, mx, false);               // began and ended in the lane
            }
            fr = __ldg(FIRST + sm.row[BLK_SPL * lane + i]);
            mn = PG_INV;
            mx = 0;
        }
        if (sl + i < s1) {
            mn = fw[i] < mn ? fw[i] : mn;
            mx = fw[i] > mx ? fw[i] : mx;
            db |= (u32)(fw[i] > fr) << i;
        }
    }
    if (DIR) {   // slot 8l+i -> bit 8(l&3)+i of word l>>2 (= slot order)
        u32 x = db << (8 * (lane & 3));
        x |= __shfl_xor_sync(0xFFFFFFFFu, x, 1);
        x |= __shfl_xor_sync(0xFFFFFFFFu, x, 2);
        if ((lane & 3) == 0) DIR[(i64)WCH_U * c + (lane >> 2)] = x;
    }
    // mn/mx: the lane's last row, open to the right; scan it across lanes
    const bool inner = (br.mb & 0xFEu) != 0;
    u32 cmn = mn, cmx = mx;
    bool started;
    blk_seg_scan(lane, hstart || inner, cmn, cmx, started);
    const u32 pmn = __shfl_up_sync(0xFFFFFFFFu, cmn, 1), pmx = __shfl_up_sync(0xFFFFFFFFu, cmx, 1);
    const bool pstarted = __shfl_up_sync(0xFFFFFFFFu, (int)started, 1) != 0 && lane > 0;
    if (inner && !hstart) {                      // head row came from the left and ends here
        const u32 tmn = lane > 0 && pmn < hmn ? pmn : hmn;
        const u32 tmx = lane > 0 && pmx > hmx ? pmx : hmx;
        write_tag(W, fh, tmn, tmx, !pstarted);
    }
    // the lane's last row ends exactly at the lane's end when the next lane starts a row
    const bool next_starts = __shfl_down_sync(0xFFFFFFFFu, (int)hstart, 1) != 0;
    if (lane < 31 && next_starts) write_tag(W, fr, cmn, cmx, !started);
    if (lane == 31) write_tag(W, fr, cmn, cmx, !started || br.last_open);
}

// --------------------------------------------------------------------------
// S4, two-level tags (large graphs).  A per-slot gather of FIRST (4 B per vertex: 1 GB at
// 2^28 vertices, 8x the L2) misses L2 on most slots and moves a 32-byte sector for 4 useful
// bytes (k_tags_blk at C5a: 137 GB of DRAM for 39 GB algorithmic).  But a row only needs its
// min and max.  So every vertex also gets a CODE of TAG_BITS bits, a monotone quantisation of
// its preorder rank (code(x) > code(y) implies x > y), packed into a table 8x (4-bit) smaller
// than FIRST that stays in L2.  Every slot looks up its target's code; the exact FIRST is
// gathered only for the slots whose code equals the row's minimum or maximum code -- about two
// per row plus a few percent of a hub row's slots.  The code boundaries are quantiles of
// first[target] over a sample of slots (denser at both ends, where a long row's extremes
// lie); they affect the number of exact gathers only, never the result.
// The direction bits become conservative: code(target) >= code(row) looks the target up
// (k_labels takes max(CID[row], CID[target]), which is right for every slot).
// --------------------------------------------------------------------------
#ifndef PG_TAG_BITS
#define PG_TAG_BITS 4
#endif
constexpr int TAG_BITS = PG_TAG_BITS;
constexpr int TAG_NB = (1 << TAG_BITS) - 1;           // boundaries; codes 0 .. TAG_NB
constexpr int TAG_PW_SH = TAG_BITS == 4 ? 3 : 2;      // log2(codes per 32-bit word)
constexpr int TAG_SAMPLES = 2048;
static_assert(TAG_BITS == 4 || TAG_BITS == 8, "codes are nibbles or bytes");

// sample position (of TAG_SAMPLES sorted values) of boundary j = 0 .. TAG_NB-1
__device__ __forceinline__ int tag_bound_pos(int j) {
    if (TAG_BITS == 8) return (j + 1) * (TAG_SAMPLES / 256);
    // 4 bits: 1/64, 1/32, 1/16, 1/8, then steps of 3/32 up to 7/8, 15/16, 31/32, 63/64
    const int U = TAG_SAMPLES / 64;
    if (j < 4) return U << j;
    if (j < 12) return 8 * U + 6 * U * (j - 3);
    return TAG_SAMPLES - (U << (14 - j));
}

// one CTA: sample slots, sort first[target], pick the boundaries
__global__ void __launch_bounds__(1024) k_tag_bounds(i64 m, const int32_t* __restrict__ tgt,
                                                      const u32* __restrict__ FIRST, u32* BND) {
    __shared__ u32 v[TAG_SAMPLES];
    for (int i = threadIdx.x; i < TAG_SAMPLES; i += 1024) {
        const u64 s = pg::sm64(0x7A65ull + (u64)i) % (u64)m;
        v[i] = __ldg(FIRST + (u32)__ldg(tgt + s));
    }
    __syncthreads();
    for (int k = 2; k <= TAG_SAMPLES; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < TAG_SAMPLES; i += 1024) {
                const int p = i ^ j;
                if (p > i) {
                    const u32 a = v[i], b = v[p];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        v[i] = b;
                        v[p] = a;
                    }
                }
            }
            __syncthreads();
        }
    if (threadIdx.x < TAG_NB) BND[threadIdx.x] = v[tag_bound_pos(threadIdx.x)];
}

// code(f) = #{j : BND[j] <= f}, packed little-endian into Q
__global__ void __launch_bounds__(256) k_tag_codes(i64 n, const u32* __restrict__ FIRST, const u32* __restrict__ BND,
                                                    u32* __restrict__ Q) {
    __shared__ u32 b[TAG_NB + 1];
    for (int i = threadIdx.x; i < TAG_NB; i += 256) b[i] = BND[i];
    if (threadIdx.x == 0) b[TAG_NB] = PG_INV;
    __syncthreads();
    constexpr int PW = 1 << TAG_PW_SH;
    const i64 wi = (i64)blockIdx.x * 256 + threadIdx.x;
    const i64 v0 = wi * PW;
    if (v0 >= n) return;
    u32 f[PW];
    if (v0 + PW <= n) {
#pragma unroll
        for (int i = 0; i < PW; i += 4) {
            const uint4 x = *reinterpret_cast<const uint4*>(FIRST + v0 + i);
            f[i] = x.x, f[i + 1] = x.y, f[i + 2] = x.z, f[i + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < PW; ++i) f[i] = v0 + i < n ? FIRST[v0 + i] : 0u;
    }
    u32 word = 0;
#pragma unroll
    for (int i = 0; i < PW; ++i) {
        u32 c = 0;   // #{j : b[j] <= f}: binary search over the sorted boundaries
#pragma unroll
        for (int st = (TAG_NB + 1) >> 1; st >= 1; st >>= 1)
            if (b[c + st - 1] <= f[i]) c += st;
        word |= c << (TAG_BITS * i);
    }
    Q[wi] = word;
}

__device__ __forceinline__ u32 tag_code(u32 word, u32 v) {
    return (word >> (TAG_BITS * (v & ((1u << TAG_PW_SH) - 1u)))) & (u32)TAG_NB;
}
// (min code, TAG_NB - max code) in the two halves of a word: one VIMNMX.U16x2 combines both
__device__ __forceinline__ u32 tag_pair(u32 c) { return c | (((u32)TAG_NB - c) << 16); }

#ifndef PG_TAGS2_MINB
#define PG_TAGS2_MINB 5
#endif
#ifndef PG_TAGS2_QL1
#define PG_TAGS2_QL1 0
#endif
#ifndef PG_TAGS2_EXACT
#define PG_TAGS2_EXACT ld_na64
#endif
__global__ void __launch_bounds__(WCH_BLOCK, PG_TAGS2_MINB) k_tags2_blk(const i64* __restrict__ off,
                                                                  const int32_t* __restrict__ tgt, i64 n, i64 m,
                                                                  const u32* __restrict__ crow,
                                                                  const u32* __restrict__ FIRST,
                                                                  const u32* __restrict__ Q, uint2* W,
                                                                  u32* __restrict__ DIR) {
    __shared__ BlkSmem smem[WCH_BLOCK / 32];
    const int lane = threadIdx.x & 31;
    const i64 c = ((i64)blockIdx.x * WCH_BLOCK + threadIdx.x) >> 5;
    if (c >= num_chunks(m)) return;
    BlkSmem& sm = smem[threadIdx.x >> 5];
    const i64 s0 = c * WCH, s1 = s0 + WCH < m ? s0 + WCH : m;
    const i64 sl = s0 + BLK_SPL * lane;
    const u32 base = crow[c];
    const i64 a_base = off[base], e_base = off[(i64)base + 1];
    const bool one_row = e_base >= s1;
    constexpr u32 NEUT = 0xFFFFFFFFu;
    u32 g[WCH_U], q[WCH_U];
    wc_load(tgt, m, c, lane, g);
    {
        const u64 pol = policy_evict_last();   // the code table stays in L2 ahead of the streams
#pragma unroll
        for (int k = 0; k < WCH_U; ++k) {
            q[k] = 0;
            if (s0 + 32 * k + lane < s1)
                q[k] = PG_TAGS2_QL1 ? ld_keep_l1(Q + (g[k] >> TAG_PW_SH), pol) : ld_keep(Q + (g[k] >> TAG_PW_SH), pol);
        }
#pragma unroll
        for (int k = 0; k < WCH_U; ++k) q[k] = tag_code(q[k], g[k]);
    }
    if (one_row) {   // warp-uniform: a hub row's chunk
        const u32 fb = __ldg(FIRST + base);
        const u32 cb = tag_code(__ldg(Q + (base >> TAG_PW_SH)), base);
        u32 x = NEUT;
#pragma unroll
        for (int k = 0; k < WCH_U; ++k)
            if (s0 + 32 * k + lane < s1) x = __vminu2(x, tag_pair(q[k]));
        u32 cmn = __reduce_min_sync(0xFFFFFFFFu, x & 0xFFFFu);
        u32 cmx = (u32)TAG_NB - __reduce_min_sync(0xFFFFFFFFu, x >> 16);
        // a minimum code above the row's own leaves w1 = first[row]; likewise the maximum
        if (cmn > cb) cmn = NEUT;
        if (cmx < cb) cmx = NEUT;
        u32 cm = 0, dw = 0;
#pragma unroll
        for (int k = 0; k < WCH_U; ++k) {
            const bool ok = s0 + 32 * k + lane < s1;
            const bool cand = ok && (q[k] == cmn || q[k] == cmx);
            if (cand) g[k] = PG_TAGS2_EXACT(FIRST + g[k]);
            cm |= (u32)cand << k;
            const unsigned b = __ballot_sync(0xFFFFFFFFu, ok && q[k] >= cb);
            if (lane == k) dw = b;
        }
        if (DIR && lane < WCH_U) DIR[(i64)WCH_U * c + lane] = dw;
        u32 mn = PG_INV, mx = 0;
#pragma unroll
        for (int k = 0; k < WCH_U; ++k)
            if (cm >> k & 1u) {
                mn = g[k] < mn ? g[k] : mn;
                mx = g[k] > mx ? g[k] : mx;
            }
        mn = __reduce_min_sync(0xFFFFFFFFu, mn);
        mx = __reduce_max_sync(0xFFFFFFFFu, mx);
        if (lane == 0 && mn != PG_INV) write_tag(W, fb, mn, mx, a_base < s0 || e_base > s1);
        return;
    }
    u32 tb[BLK_SPL];
    blk_transpose(sm, lane, g, tb);
    uint2 cw;
    {   // the codes take the same way, as bytes
        __syncwarp();
        uint8_t* cbuf = reinterpret_cast<uint8_t*>(sm.xp);
#pragma unroll
        for (int k = 0; k < WCH_U; ++k) cbuf[32 * k + lane] = (uint8_t)q[k];
        __syncwarp();
        cw = *reinterpret_cast<const uint2*>(cbuf + BLK_SPL * lane);
    }
    const BlkRows br = blk_rows(off, n, s0, s1, base, lane, sm);
    const bool hstart = br.mb & 1u;
    // (min, max) code of every row of the chunk, known to each of its slots: the lane's own
    // pass, then a forward and a backward segmented scan over the lanes
    u32 ci[BLK_SPL], fw[BLK_SPL];
    u32 head = NEUT;
    {
        u32 acc = NEUT;
        bool seen = false;
#pragma unroll
        for (int i = 0; i < BLK_SPL; ++i) {
            ci[i] = ((i < 4 ? cw.x >> (8 * i) : cw.y >> (8 * (i - 4))) & 0xFFu);
            if (br.mb >> i & 1u) {
                if (!seen) head = acc;
                seen = true;
                acc = NEUT;
            }
            if (sl + i < s1) acc = __vminu2(acc, tag_pair(ci[i]));
        }
        if (!seen) head = acc;
        fw[BLK_SPL - 1] = acc;   // the lane's last (open) row
    }
    const unsigned hb = __ballot_sync(0xFFFFFFFFu, br.mb != 0u);
    u32 F = fw[BLK_SPL - 1], Bk = head;
    {
        const unsigned le = lane == 31 ? 0xFFFFFFFFu : (2u << lane) - 1u;
        const int lo = (hb & le) ? 31 - __clz(hb & le) : 0;
        const unsigned ge = hb >> lane;
        const int hi = ge ? lane + __ffs(ge) - 1 : 31;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 a = __shfl_up_sync(0xFFFFFFFFu, F, o);
            const u32 b = __shfl_down_sync(0xFFFFFFFFu, Bk, o);
            if (lane - o >= lo) F = __vminu2(F, a);
            if (lane + o <= hi) Bk = __vminu2(Bk, b);
        }
    }
    u32 Fprev = __shfl_up_sync(0xFFFFFFFFu, F, 1), Bnext = __shfl_down_sync(0xFFFFFFFFu, Bk, 1);
    if (lane == 0) Fprev = NEUT;
    if (lane == 31) Bnext = NEUT;
    {
        u32 acc = Fprev;
#pragma unroll
        for (int i = 0; i < BLK_SPL; ++i) {
            if (br.mb >> i & 1u) acc = NEUT;
            if (sl + i < s1) acc = __vminu2(acc, tag_pair(ci[i]));
            fw[i] = acc;
        }
    }
    u32 cm = 0;
    {
        u32 full = __vminu2(fw[BLK_SPL - 1], Bnext);
#pragma unroll
        for (int i = BLK_SPL - 1; i >= 0; --i) {
            if (i < BLK_SPL - 1 && (br.mb >> (i + 1) & 1u)) full = fw[i];
            const bool cand = sl + i < s1 && (ci[i] == (full & 0xFFFFu) || (u32)TAG_NB - ci[i] == (full >> 16));
            cm |= (u32)cand << i;
        }
    }
#pragma unroll
    for (int i = 0; i < BLK_SPL; ++i)
        if (cm >> i & 1u) tb[i] = PG_TAGS2_EXACT(FIRST + tb[i]);
    // from here on as k_tags_blk, over the candidates only
    const u32 fh = __ldg(FIRST + br.r_first);
    u32 fr = fh;
    u32 rc = tag_code(__ldg(Q + (br.r_first >> TAG_PW_SH)), br.r_first);
    u32 mn = PG_INV, mx = 0, hmn = PG_INV, hmx = 0, db = 0;
    bool in_head = true;
#pragma unroll
    for (int i = 0; i < BLK_SPL; ++i) {
        if (i > 0 && (br.mb >> i & 1u)) {
            if (in_head) {
                hmn = mn;
                hmx = mx;
                in_head = false;
                if (hstart) write_tag(W, fr, mn, mx, false);
            } else {
                write_tag(W, fr, mn, mx, false);
            }
            const u32 r = sm.row[BLK_SPL * lane + i];
            fr = __ldg(FIRST + r);
            rc = tag_code(__ldg(Q + (r >> TAG_PW_SH)), r);
            mn = PG_INV;
            mx = 0;
        }
        if (cm >> i & 1u) {
            mn = tb[i] < mn ? tb[i] : mn;
            mx = tb[i] > mx ? tb[i] : mx;
        }
        if (sl + i < s1) db |= (u32)(ci[i] >= rc) << i;
    }
    if (DIR) {
        u32 x = db << (8 * (lane & 3));
        x |= __shfl_xor_sync(0xFFFFFFFFu, x, 1);
        x |= __shfl_xor_sync(0xFFFFFFFFu, x, 2);
        if ((lane & 3) == 0) DIR[(i64)WCH_U * c + (lane >> 2)] = x;
    }
    const bool inner = (br.mb & 0xFEu) != 0;
    u32 cmn = mn, cmx = mx;
    bool started;
    blk_seg_scan(lane, hstart || inner, cmn, cmx, started);
    const u32 pmn = __shfl_up_sync(0xFFFFFFFFu, cmn, 1), pmx = __shfl_up_sync(0xFFFFFFFFu, cmx, 1);
    const bool pstarted = __shfl_up_sync(0xFFFFFFFFu, (int)started, 1) != 0 && lane > 0;
    if (inner && !hstart) {
        const u32 tmn = lane > 0 && pmn < hmn ? pmn : hmn;
        const u32 tmx = lane > 0 && pmx > hmx ? pmx : hmx;
        write_tag(W, fh, tmn, tmx, !pstarted);
    }
    const bool next_starts = __shfl_down_sync(0xFFFFFFFFu, (int)hstart, 1) != 0;
    if (lane < 31 && next_starts) write_tag(W, fr, cmn, cmx, !started);
    if (lane == 31) write_tag(W, fr, cmn, cmx, !started || br.last_open);
}

// --------------------------------------------------------------------------
// S4: low/high by a blocked sparse table over preorder positions (32-wide blocks)
// --------------------------------------------------------------------------
__device__ __forceinline__ uint2 mm(uint2 a, uint2 b) {
    return make_uint2(a.x < b.x ? a.x : b.x, a.y > b.y ? a.y : b.y);
}
__device__ __forceinline__ uint2 shfl_down2(uint2 v, int o) {
    return make_uint2(__shfl_down_sync(0xFFFFFFFFu, v.x, o), __shfl_down_sync(0xFFFFFFFFu, v.y, o));
}
__device__ __forceinline__ uint2 shfl_up2(uint2 v, int o) {
    return make_uint2(__shfl_up_sync(0xFFFFFFFFu, v.x, o), __shfl_up_sync(0xFFFFFFFFu, v.y, o));
}
__device__ __forceinline__ uint2 shfl_idx2(uint2 v, int src) {
    return make_uint2(__shfl_sync(0xFFFFFFFFu, v.x, src), __shfl_sync(0xFFFFFFFFu, v.y, src));
}

// Positions [0, niso) are the isolated vertices' slots: no query range reaches them (a tree's
// positions are contiguous and lie above), so their blocks are skipped and they enter the
// boundary block as neutral elements.
__global__ void k_rmq_block(i64 n, const uint2* __restrict__ W, uint2* PM, uint2* ST0, const Ctr* ctr) {
    const i64 niso = ctr->niso;
    if (((i64)blockIdx.x + 1) * blockDim.x <= niso) return;
    i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    int lane = threadIdx.x & 31;
    uint2 v = i < n && i >= niso ? W[i] : make_uint2(PG_INV, 0u);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint2 u = shfl_up2(v, o);
        if (lane >= o) v = mm(v, u);
    }
    if (i < n) PM[i] = v;
    if (lane == 31 && (i >> 5) < cdiv(n, 32)) ST0[i >> 5] = v;
}

__global__ void k_rmq_level(i64 nb, const uint2* __restrict__ src, uint2* dst, i64 half, const Ctr* ctr) {
    i64 b = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb || b < ((i64)ctr->niso >> 5) - 8) return;   // entries below the isolated slots' end are never read
    uint2 v = src[b];
    if (b + half < nb) v = mm(v, src[b + half]);
    dst[b] = v;
}

// every level of the sparse table in one CTA (small graphs: 11-15 launches otherwise)
constexpr i64 RMQ_SMALL = 1 << 16;
__global__ void __launch_bounds__(1024) k_rmq_levels_small(i64 nb, i64 lv, uint2* ST) {
    for (i64 k = 1; k < lv; ++k) {
        const uint2* src = ST + (k - 1) * nb;
        uint2* dst = ST + k * nb;
        const i64 half = (i64)1 << (k - 1);
        for (i64 b = threadIdx.x; b < nb; b += blockDim.x) {
            uint2 v = src[b];
            if (b + half < nb) v = mm(v, src[b + half]);
            dst[b] = v;
        }
        __syncthreads();
    }
}

// low/high of every preorder position, fence test, and Last-CC union of the non-fence
// tree edges (S5 fused).
__global__ void k_rmq_query(i64 n, const uint2* __restrict__ W, const u32* __restrict__ E,
                            const u32* __restrict__ PV, const u32* __restrict__ PPAR,
                            const uint2* __restrict__ PM, const uint2* __restrict__ ST, i64 nb,
                            const uint2* __restrict__ FL, u32* FPF, const Ctr* ctr) {
    i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const i64 niso = ctr->niso;
    if (i - lane + 32 <= niso) {     // warp-uniform: isolated slots only (each its own root)
        if (i < n) FPF[i] = PG_INV;
        return;
    }
    const bool valid = i < n;
    uint2 w = valid && i >= niso ? W[i] : make_uint2(PG_INV, 0u);
    u32 e = valid && i >= niso ? E[i] : (u32)i;
    // in-register doubling table over [lane, lane + 2^k) within the 32-block
    uint2 M[6];
    M[0] = w;
#pragma unroll
    for (int k = 1; k < 6; ++k) {
        int h = 1 << (k - 1);
        uint2 o = shfl_down2(M[k - 1], h);
        M[k] = lane + h < 32 ? mm(M[k - 1], o) : M[k - 1];
    }
    uint2 sfx = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint2 u = shfl_down2(sfx, o);
        if (lane + o < 32) sfx = mm(sfx, u);
    }
    const u64 bi = (u64)i >> 5, be = (u64)e >> 5;
    const bool inblock = be == bi;
    int kq = 0, src = lane;
    if (inblock) {
        u32 len = e - (u32)i + 1;
        kq = 31 - __clz(len);
        src = (int)(e & 31) - (1 << kq) + 1;
    }
    uint2 mine = M[0], far = M[0];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        uint2 t = shfl_idx2(M[k], k == kq ? src : lane);
        if (k == kq) {
            far = t;
            mine = M[k];
        }
    }
    if (!valid) return;
    uint2 res;
    if (inblock) {
        res = mm(mine, far);
    } else {
        res = mm(sfx, PM[e]);
        if (be > bi + 1) {
            u64 l = bi + 1, r = be - 1;
            u64 len = r - l + 1;
            int k = 63 - __clzll((long long)len);
            const uint2* lvl = ST + (i64)k * nb;
            res = mm(res, mm(lvl[l], lvl[r - ((u64)1 << k) + 1]));
        }
    }
    u32 fpf = PG_INV;
    u32 v = 0, p = 0;
    if (i >= niso) v = PV[i], p = PPAR[i];
    if (p != v) {
        uint2 fp = FL[p];
        bool fence = fp.x <= res.x && res.y <= fp.y;
        fpf = fp.x | (fence ? 0x80000000u : 0u);  // non-fence tree edges: k_cc2_local / _tree
    }
    FPF[i] = fpf;
}

// --------------------------------------------------------------------------
// S5: Last-CC over cross edges.  Sampling first (Afforest): every position links the cross
// edge its high tag points at (k_cc2_local / k_cc2_links), so the big skeleton component forms before
// the sampled-giant rows are skipped by the full pass.  It replaced sampling the last two
// slots of each row (two random (first, last) gathers per vertex): C5a Last-CC 18.2 ->
// 12.8 ms, C4 4.4 -> 3.2, C3 1.6 -> 1.4, C2 0.81 -> 0.48.
// --------------------------------------------------------------------------
__device__ __forceinline__ bool is_cross(uint2 fu, uint2 fw) {
    return !((fu.x <= fw.x && fw.x <= fu.y) || (fw.x <= fu.x && fu.x <= fw.y));
}

// Last-CC links preorder positions, so every skeleton component's union-find root is the
// preorder rank of its head (the component's minimum).
// Last-CC local phase over preorder positions: non-fence tree edges (i, parent position)
// inside a block of LOCAL_B positions are joined in shared memory (a child's parent is
// usually a few positions back), then C[i] = block root is published.
__global__ void __launch_bounds__(LOCAL_T) k_cc2_local(i64 n, int lb, const u32* __restrict__ FPF,
                                                       const uint2* __restrict__ W, const u32* __restrict__ E, u32* C,
                                                       const Ctr* ctr) {
    __shared__ u32 sp[LOCAL_B];
    const i64 b0 = (i64)blockIdx.x << lb;
    const int cnt = (int)(n - b0 < (1 << lb) ? n - b0 : (1 << lb));
    const i64 niso = ctr->niso;
    if (b0 + cnt <= niso) {       // isolated slots only: singletons, nothing to read
        for (int i = threadIdx.x; i < cnt; i += LOCAL_T) C[b0 + i] = (u32)(b0 + i);
        return;
    }
    for (int i = threadIdx.x; i < cnt; i += LOCAL_T) sp[i] = (u32)i;
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += LOCAL_T) {
        if (b0 + i < niso) continue;
        u32 f = FPF[b0 + i];
        {     // the high tag's cross edge (k_cc2_links), when it stays in the block
            const u32 hi = __ldcs(&W[b0 + i].y);
            if (hi > __ldcs(E + b0 + i) && (i64)hi < b0 + (1 << lb)) slink(sp, (u32)i, (u32)(hi - b0));
        }
        if (f & 0x80000000u) continue;     // fence, or a root (PG_INV)
        if ((i64)f >= b0) slink(sp, (u32)i, (u32)(f - b0));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += LOCAL_T) C[b0 + i] = (u32)b0 + sfind(sp, (u32)i);
}

// Sampling without gathers: the high tag w2[i] (before the RMQ) is the
// largest preorder rank among the neighbours of the vertex at position i.  When it lies
// beyond the vertex's subtree (w2 > last) that neighbour is neither a descendant nor an
// ancestor, so the edge is a cross edge of the skeleton: link it.  One coalesced read of W
// and E per position replaces two random (first, last) gathers per vertex.
//
// Both block-crossing global links of a position in one pass: its non-fence tree edge and
// the cross edge of its high tag (a cross edge never points into its own subtree, so
// hi > last >= i and a block-local one was taken by k_cc2_local).
__global__ void k_cc2_links(i64 n, int lb, const u32* __restrict__ FPF, const uint2* __restrict__ W,
                            const u32* __restrict__ E, u32* C, const Ctr* ctr) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || i < (i64)ctr->niso) return;
    const u32 f = FPF[i];
    const u32 hi = __ldcs(&W[i].y);
    const u32 e = __ldcs(E + i);
    const bool tree = !(f & 0x80000000u) && (f >> lb) != (u32)(i >> lb);
    const bool cross = hi > e && (hi >> lb) != (u32)(i >> lb);
    if (tree) uf_link(C, (u32)i, f);
    if (cross) uf_link(C, (u32)i, hi);
}

// over preorder positions i (vertex PV[i]); tree roots have only back edges (every vertex
// of the tree descends from the root), so they are skipped
__global__ void k_cc2_rest(i64 n, const i64* __restrict__ off, const int32_t* __restrict__ tgt,
                           const uint2* __restrict__ FL, const u32* __restrict__ PV, const u32* __restrict__ E,
                           const u32* __restrict__ P, u32* C, Ctr* ctr, u32* heavy) {
    i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || i < (i64)ctr->niso || ldcg(C + i) == ctr->giant2) return;
    u32 u = PV[i];
    if (P[u] == u) return;
    i64 a = off[u], b = off[u + 1];
    if (b - a < 2) return;
    if (b - a > HEAVY_ROW) {
        queue_heavy(n, b - a, u, heavy, &ctr->nheavy2, &ctr->nvheavy2);
        return;
    }
    uint2 fu = make_uint2((u32)i, E[i]);
    // 4 slots at a time: their target loads, then their (first, last) gathers, in flight together
    for (i64 s = a; s < b; s += 4) {
        u32 w[4];
        uint2 fw[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = s + k < b ? (u32)tgt[s + k] : (u32)u;
#pragma unroll
        for (int k = 0; k < 4; ++k) fw[k] = FL[w[k]];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (s + k < b && is_cross(fu, fw[k])) uf_link(C, (u32)i, fw[k].x);
    }
}

__global__ void k_cc2_rest_heavy(i64 n, const i64* __restrict__ off, const int32_t* __restrict__ tgt,
                                 const uint2* __restrict__ FL, u32* C, const Ctr* ctr, const u32* __restrict__ heavy) {
    const u32 nh = ctr->nheavy2, nvh = ctr->nvheavy2;
    for (u32 h = blockIdx.x; h < nh; h += gridDim.x) {
        u32 u = heavy[h];
        uint2 fu = FL[u];
        for (i64 s = off[u] + threadIdx.x; s < off[u + 1]; s += blockDim.x) {
            const int32_t w = tgt[s];
            if (s > off[u] && tgt[s - 1] == w) continue;
            uint2 fw = FL[(u32)w];
            if (is_cross(fu, fw)) uf_link(C, fu.x, fw.x);
        }
    }
    for (u32 h = 0; h < nvh; ++h) {
        u32 u = heavy[n - 1 - h];
        uint2 fu = FL[u];
        for (i64 s = off[u] + (i64)blockIdx.x * blockDim.x + threadIdx.x; s < off[u + 1];
             s += (i64)gridDim.x * blockDim.x) {
            const int32_t w = tgt[s];
            if (s > off[u] && tgt[s - 1] == w) continue;
            uint2 fw = FL[(u32)w];
            if (is_cross(fu, fw)) uf_link(C, fu.x, fw.x);
        }
    }
}

// final roots over positions + component count
__global__ void __launch_bounds__(256, PG_CMP_MINB) k_compress_final(i64 n, u32* C, Ctr* ctr) {
    u32 root[COMPRESS_ILP2];
    i64 idx[COMPRESS_ILP2];
    compress_ilp<COMPRESS_ILP2>(n, C, root, idx, (i64)ctr->niso);
    u32 cnt = 0;
#pragma unroll
    for (int j = 0; j < COMPRESS_ILP2; ++j) cnt += __popc(__ballot_sync(0xFFFFFFFFu, idx[j] < n && root[j] == (u32)idx[j]));
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&ctr->ncomp, cnt);
}

// --------------------------------------------------------------------------
// S6: articulation points, labels, count
// --------------------------------------------------------------------------
// articulation, in preorder space (position i = first[v]): every vertex whose tree edge is
// a fence and whose skeleton component differs from its parent's heads a BCC hanging off
// the parent; a non-root parent is then an articulation point, a root only if its head
// children span >= 2 components.  P (First-CC) has P[x] == x exactly at tree roots.
// Hubs: siblings with small subtrees sit at adjacent positions, so a warp first groups runs
// of adjacent lanes with one parent (one update per run; two components within a run
// already decide a root), and the bit and
// the write-once ROOTMARK are read before any atomic -- a 33M-leaf star otherwise spent
// 21 ms in same-address atomics on the hub.
__global__ void k_artic(i64 n, const u32* __restrict__ PPAR, const u32* __restrict__ FPF, const u32* __restrict__ C,
                        const u32* __restrict__ P, u32* ROOTMARK, u32* bits, const Ctr* ctr) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const u32 niso = ctr->niso;
    if (((i64)blockIdx.x + 1) * blockDim.x <= (i64)niso) return;   // isolated slots: no tree edge
    const int lane = threadIdx.x & 31;
    bool head = false;
    u32 p = PG_INV, ci = 0;
    if (i < n && i >= (i64)niso) {
        const u32 f = FPF[i];
        if (f != PG_INV && (f & 0x80000000u)) {
            ci = C[i];
            if (ci != C[f & 0x7FFFFFFFu]) {      // fence child inside p's own component: not a head
                head = true;
                p = PPAR[i];
            }
        }
    }
    const unsigned hm = __ballot_sync(0xFFFFFFFFu, head);
    if (!hm) return;                                         // warp-uniform
    // groups = runs of adjacent head lanes with one parent (star leaves are adjacent)
    const u32 pp = __shfl_up_sync(0xFFFFFFFFu, p, 1), pc = __shfl_up_sync(0xFFFFFFFFu, ci, 1);
    const bool cont = head && lane > 0 && (hm >> (lane - 1) & 1u) && pp == p;
    const unsigned lead = hm & ~__ballot_sync(0xFFFFFFFFu, cont);        // first lane of each run
    const unsigned mism = __ballot_sync(0xFFFFFFFFu, cont && pc != ci);   // run spans >= 2 components
    if (!(lead >> lane & 1u)) return;
    const unsigned after = lead & ~((2u << lane) - 1u);                  // later run leaders
    const unsigned run = (after ? (1u << (__ffs(after) - 1)) : 0u) - (1u << lane);   // this run's lanes
    const bool differ = (mism & (after ? run : ~((1u << lane) - 1u))) != 0;
    const u32 bit = 1u << (p & 31);
    if (*(volatile u32*)(bits + (p >> 5)) & bit) return;    // already an articulation point
    if (P[p] != p || differ) {
        atomicOr(bits + (p >> 5), bit);
        return;
    }
    u32 cur = *(volatile u32*)(ROOTMARK + p);               // write-once: PG_INV -> first head's cid
    if (cur == PG_INV) cur = atomicCAS(ROOTMARK + p, PG_INV, ci);
    if (cur != PG_INV && cur != ci) atomicOr(bits + (p >> 5), bit);
}

// per vertex (coalesced): CIDV[v] = component of position first[v] (one random read of the
// compressed C), plus the giant component's membership bitmap (one ballot per word)
__global__ void k_cid_vertices(i64 n, const u32* __restrict__ C, const u32* __restrict__ FIRST, Ctr* ctr, u32* CIDV,
                               u32* GBIT, u32* out_comp) {
    i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const u32 g = C[ctr->giant2];        // C is fully compressed: the root of the sampled giant
    if (v == 0) ctr->gcid = g;
    u32 cid = PG_INV;
    if (v < n) {
        const u32 f = __ldg(FIRST + v);
        cid = f < ctr->niso ? f : __ldg(C + f);   // an isolated vertex is its own component
        CIDV[v] = cid;
        if (out_comp) out_comp[v] = cid;
    }
    unsigned b = __ballot_sync(0xFFFFFFFFu, cid == g);
    if ((threadIdx.x & 31) == 0 && v < n) GBIT[v >> 5] = b;
}

// label(u,w) = component of the endpoint with the larger preorder rank (results.py:80-87).
// With component ids = preorder rank of the component's head this is max(CID[u], CID[w]):
// for a tree or back edge (a ancestor of d), either both share d's component or a is the
// parent of d's component head, whose rank exceeds a's and hence a's component id; a
// cross edge joins one component.  Most slots of a power-law graph point into the giant
// component, so the target's component comes from the L2-resident membership bitmap and
// only the remaining slots gather CIDV from HBM.
#ifndef PG_LABELS_HALVES
#define PG_LABELS_HALVES 8
#endif
#ifndef PG_LABELS_ONEROW
#define PG_LABELS_ONEROW 4   // windows in flight together; 0: off (C5a labels 16.1 -> 14.9 ms; 8: 15.6)
#endif
#ifndef PG_LABELS_GATHER
#define PG_LABELS_GATHER ld_na64
#endif
__global__ void __launch_bounds__(WCH_BLOCK, PG_LABELS_MINB) k_labels(const i64* __restrict__ off, const int32_t* __restrict__ tgt,
                                                      i64 n, i64 m, const u32* __restrict__ crow,
                                                      const u32* __restrict__ CIDV, const u32* __restrict__ GBIT,
                                                      const Ctr* __restrict__ ctr, const u32* __restrict__ DIR,
                                                      u32* label) {
    const int lane = threadIdx.x & 31;
    const i64 c = ((i64)blockIdx.x * WCH_BLOCK + threadIdx.x) >> 5;
    if (c >= num_chunks(m)) return;
    const i64 s0 = c * WCH, s1 = s0 + WCH < m ? s0 + WCH : m;
    const u32 g = ctr->gcid;
    u32 w[WCH_U];
#pragma unroll
    for (int k = 0; k < WCH_U; ++k) {
        i64 s = s0 + 32 * k + lane;
        w[k] = s < s1 ? (u32)__ldcs(tgt + s) : 0u;
    }
    // direction bits from k_tags_blk: a slot whose target lies earlier in preorder takes its
    // row's component (the row is the deeper endpoint), so only the other half looks up
    // the target (without DIR every slot does)
    u32 dmask = 0xFFFFFFFFu;
    if (DIR) dmask = __ldcs(DIR + (i64)WCH_U * c + (lane & (WCH_U - 1)));
    u32 cur = crow[c];
#if PG_LABELS_ONEROW
    // One (hub) row over the whole chunk -- most slots of a power-law graph: no row search, and
    // every window's lookups are in flight together: two dependent memory phases per chunk
    // (bitmap, then the non-giant targets' CIDV) instead of two per window, which is what the
    // kernel waits on
    if (off[(i64)cur + 1] >= s1) {   // warp-uniform
        const u32 cu = __ldg(CIDV + cur);
        constexpr int OW = PG_LABELS_ONEROW;   // windows in flight together
#pragma unroll
        for (int h = 0; h < WCH_U; h += OW) {
            u32 cw[OW];
            u32 look = 0;
#pragma unroll
            for (int k = 0; k < OW; ++k) {
                const u32 dwk = __shfl_sync(0xFFFFFFFFu, dmask, h + k);
                const bool lk = s0 + 32 * (h + k) + lane < s1 && ((dwk >> lane) & 1u);
                look |= (u32)lk << k;
                cw[k] = lk ? __ldg(GBIT + (w[h + k] >> 5)) : 0u;
            }
#pragma unroll
            for (int k = 0; k < OW; ++k)
                cw[k] = !(look >> k & 1u) ? 0u : (cw[k] >> (w[h + k] & 31)) & 1u ? g : PG_LABELS_GATHER(CIDV + w[h + k]);
#pragma unroll
            for (int k = 0; k < OW; ++k) {
                const i64 s = s0 + 32 * (h + k) + lane;
                if (s < s1) {
                    u32 lab = cu > cw[k] ? cu : cw[k];
                    if (w[h + k] == cur) lab = PG_INV;
                    __stcs(label + s, lab);
                }
            }
        }
        return;
    }
#endif
    // the chunk in PG_LABELS_HALVES parts: fewer live registers (32 per thread, no spills)
    constexpr int H = WCH_U / PG_LABELS_HALVES;
#pragma unroll
    for (int h = 0; h < WCH_U; h += H) {
        u32 cw[H], rw[H];
        // rows of the part's windows first: the offset loads and shuffles overlap the gathers
#pragma unroll
        for (int k = 0; k < H; ++k) {
            rw[k] = 0;
            const i64 sb = s0 + 32 * (h + k);
            if (sb < s1) {   // warp-uniform
                rw[k] = wc_resolve_row(off, n, cur, sb, lane, sb + lane < s1);
                cur = __shfl_sync(0xFFFFFFFFu, rw[k], 31);
            }
        }
        u32 look = 0;
#pragma unroll
        for (int k = 0; k < H; ++k) {
            i64 s = s0 + 32 * (h + k) + lane;
            // every lane takes part in the shuffle (a short-circuited one leaves the source
            // lane out in the last, partial window)
            const u32 dwk = __shfl_sync(0xFFFFFFFFu, dmask, h + k);
            const bool lk = s < s1 && ((dwk >> lane) & 1u);
            look |= (u32)lk << k;
            cw[k] = lk ? __ldg(GBIT + (w[h + k] >> 5)) : 0u;
        }
#pragma unroll
        for (int k = 0; k < H; ++k) {
            cw[k] = !(look >> k & 1u) ? 0u : (cw[k] >> (w[h + k] & 31)) & 1u ? g : PG_LABELS_GATHER(CIDV + w[h + k]);
        }
#pragma unroll
        for (int k = 0; k < H; ++k) {
            const i64 s = s0 + 32 * (h + k) + lane;
            if (s >= s1) break;
            u32 cu = __ldg(CIDV + rw[k]);
            u32 lab = cu > cw[k] ? cu : cw[k];
            if (w[h + k] == rw[k]) lab = PG_INV;  // self-loop: unlabelled, as in the reference (-1)
            __stcs(label + s, lab);
        }
    }
}

// every tree root (isolated vertices included) is a singleton skeleton component
__global__ void k_finish(const Ctr* ctr, i64* bcc_count) {
    *bcc_count = (i64)ctr->ncomp - (i64)ctr->r1 - (i64)ctr->niso;
}

// --------------------------------------------------------------------------
// canonical labels: min undirected edge id per BCC (results.py:103-112 equivalent)
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(WCH_BLOCK) k_canon_count(const i64* __restrict__ off, const int32_t* __restrict__ tgt,
                                                           i64 n, i64 m, const u32* __restrict__ crow, u32* UCNT) {
    const int lane = threadIdx.x & 31;
    const i64 c = ((i64)blockIdx.x * WCH_BLOCK + threadIdx.x) >> 5;
    if (c >= num_chunks(m)) return;
    const i64 s0 = c * WCH, s1 = s0 + WCH < m ? s0 + WCH : m;
    u32 cur = crow[c];
#pragma unroll 1
    for (i64 sb = s0; sb < s1; sb += 32) {
        const i64 s = sb + lane;
        const bool valid = s < s1;
        const unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
        const u32 row = wc_resolve_row(off, n, cur, sb, lane, valid);
        cur = __shfl_sync(0xFFFFFFFFu, row, 31);
        const Seg g = wc_segment(row, lane, valid, vm);
        if (valid) {
            u32 up = (u32)tgt[s] > row ? 1u : 0u;
            u32 cnt = __reduce_add_sync(g.mask, up);
            if (lane == g.lo && cnt) {
                if (!g.cut_left && !g.cut_right) UCNT[row] = cnt;
                else atomicAdd(UCNT + row, cnt);
            }
        }
    }
}

__global__ void __launch_bounds__(WCH_BLOCK) k_canon_min(const i64* __restrict__ off, const int32_t* __restrict__ tgt,
                                                         i64 n, i64 m, const u32* __restrict__ crow,
                                                         const u32* __restrict__ UCNT, const u32* __restrict__ UOFF,
                                                         const u32* __restrict__ label, i64 nlab, u32* CANON) {
    const int lane = threadIdx.x & 31;
    const i64 c = ((i64)blockIdx.x * WCH_BLOCK + threadIdx.x) >> 5;
    if (c >= num_chunks(m)) return;
    const i64 s0 = c * WCH, s1 = s0 + WCH < m ? s0 + WCH : m;
    u32 cur = crow[c];
#pragma unroll 1
    for (i64 sb = s0; sb < s1; sb += 32) {
        const i64 s = sb + lane;
        const bool valid = s < s1;
        const u32 row = wc_resolve_row(off, n, cur, sb, lane, valid);
        cur = __shfl_sync(0xFFFFFFFFu, row, 31);
        bool up = false;
        u32 lab = 0, eid = 0;
        if (valid && (u32)tgt[s] > row) {
            // the row's upper part is its last UCNT slots (rows are sorted)
            eid = (u32)((i64)UOFF[row] + (s - (off[row + 1] - (i64)UCNT[row])));
            lab = label[s];
            up = (i64)lab < nlab;   // ids outside [0, nlab) are not canonicalised
        }
        unsigned act = __ballot_sync(0xFFFFFFFFu, up);
        if (up) {
            unsigned grp = __match_any_sync(act, lab);
            // slots are in CSR order, so the lowest lane of a group carries its min eid
            if (lane == __ffs(grp) - 1 && __ldcg(CANON + lab) > eid) atomicMin(CANON + lab, eid);
        }
    }
}

__global__ void k_canon_apply(i64 m, const u32* __restrict__ CANON, i64 nlab, const u32* in, u32* out) {
    i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m) return;
    u32 l = in[s];
    out[s] = (i64)l < nlab ? CANON[l] : l;
}

struct UcntLoad {
    const u32* UCNT;
    __device__ __forceinline__ u32 operator()(i64 i) const { return UCNT[i]; }
};
struct UoffStore {
    u32* UOFF;
    __device__ __forceinline__ void operator()(i64 i, u32 ex, u32) const { UOFF[i] = ex; }
};

// --------------------------------------------------------------------------
// validation (graph.py:87-107 ranges, graph.py:123-158 symmetry, SPEC.md:457 simple)
// --------------------------------------------------------------------------
constexpr u32 VERR_RANGE = 1, VERR_UNSORTED = 2, VERR_NOTSYM = 4;

__global__ void k_validate_offsets(i64 n, i64 m, const i64* __restrict__ off, Ctr* ctr) {
    i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (v > n) return;
    bool bad = false;
    if (v == 0 && off[0] != 0) bad = true;
    if (v == n && off[n] != m) bad = true;
    if (v < n && off[v] > off[v + 1]) bad = true;
    if (bad) atomicOr(&ctr->verr, VERR_RANGE);
}

__device__ __forceinline__ i64 lower_bound_row(const int32_t* tgt, i64 a, i64 b, int32_t key) {
    while (a < b) {
        i64 mid = (a + b) >> 1;
        if (tgt[mid] < key) a = mid + 1; else b = mid;
    }
    return a;
}

// Exact multiset symmetry, bucketed so that every search is cache-local.
//
// Slots split into "up" (u -> w, w > u), "down" (w < u) and self-loops.  A maximal run of c
// equal up slots u -> w in row u becomes one key (w, u, c > 1); the graph is symmetric iff
// every key finds exactly c copies of u in row w and #up == #down (runs are distinct pairs,
// so the key -> run map is injective on down slots, and equal counts make it onto).
//   k_val_pass<false>  streams the CSR: range / order checks, up & down counts, and a
//                      per-block histogram of the keys' bucket (w >> shift, VAL_BINS);
//   (host)             rejects #up != #down before any key is written (so keys <= m/2);
//   launch_scan        bucket-major exclusive scan of the histograms -> per-block bases;
//   k_val_pass<true>   re-streams the same chunks and scatters the keys into buckets;
//   k_val_check        walks the keys bucket by bucket, so the rows it searches (a
//                      1/VAL_BINS slice of the id range) stay resident in L2.
// The first version searched row w straight from the slot pass: ~17 DRAM sectors per
// search on RMAT 2^28 (ncu: 1.17 TB read, 291 ms); searching the shorter row instead
// still took 246 ms, because every slot then gathers the other row's offsets.
constexpr int VAL_BINS_LB = 10, VAL_BINS = 1 << VAL_BINS_LB;
constexpr int VAL_GRID = 148 * 8;
constexpr u64 VAL_DUP = 1ull << 63;

template <bool SCATTER>
__global__ void __launch_bounds__(WCH_BLOCK) k_val_pass(const i64* __restrict__ off, const int32_t* __restrict__ tgt,
                                                        i64 n, i64 m, const u32* __restrict__ crow, int shift,
                                                        Ctr* ctr, unsigned long long* cnt, u32* hist,
                                                        const u32* __restrict__ base, u64* __restrict__ keys) {
    __shared__ u32 s_bin[VAL_BINS];
    if (SCATTER && cnt[0] != cnt[1]) return;   // unbalanced: failed already, and keys could exceed m/2
    for (int i = threadIdx.x; i < VAL_BINS; i += WCH_BLOCK)
        s_bin[i] = SCATTER ? base[(i64)i * gridDim.x + blockIdx.x] : 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const i64 nch = num_chunks(m);
    const i64 stride = (i64)gridDim.x * (WCH_BLOCK / 32);
    u32 err = 0, nup = 0, ndown = 0, nkey = 0;
#pragma unroll 1
    for (i64 c = ((i64)blockIdx.x * WCH_BLOCK + threadIdx.x) >> 5; c < nch; c += stride) {
        const i64 s0 = c * WCH, s1 = s0 + WCH < m ? s0 + WCH : m;
        u32 cur = crow[c];
#pragma unroll 1
        for (i64 sb = s0; sb < s1; sb += 32) {
            const i64 s = sb + lane;
            const bool valid = s < s1;
            const u32 row = wc_resolve_row(off, n, cur, sb, lane, valid);
            cur = __shfl_sync(0xFFFFFFFFu, row, 31);
            bool key = false;
            u32 bin = PG_INV;
            u64 kv = 0;
            if (valid) {
                const i64 u = row;
                const int32_t w = tgt[s];
                if (!SCATTER && (w < 0 || (i64)w >= n)) {
                    err |= VERR_RANGE;
                } else {
                    const i64 rs = off[u], re = off[u + 1];
                    if (!SCATTER && s + 1 < re && tgt[s + 1] < w) err |= VERR_UNSORTED;
                    if ((i64)w > u) {
                        ++nup;
                        if (s == rs || tgt[s - 1] != w) {            // first slot of its run
                            key = true;
                            bin = (u32)w >> shift;
                            const bool dup = s + 1 < re && tgt[s + 1] == w;
                            kv = (dup ? VAL_DUP : 0ull) | ((u64)(u32)w << 32) | (u64)(u32)u;
                        }
                    } else if ((i64)w < u) {
                        ++ndown;
                    }
                }
            }
            if (__ballot_sync(0xFFFFFFFFu, key)) {
                const unsigned peers = __match_any_sync(0xFFFFFFFFu, bin);   // key lanes by bucket
                if (key) {
                    ++nkey;
                    const int leader = __ffs(peers) - 1;
                    u32 b0 = 0;
                    if (lane == leader) b0 = atomicAdd(&s_bin[bin], (u32)__popc(peers));
                    if (SCATTER) {
                        b0 = __shfl_sync(peers, b0, leader);
                        keys[b0 + (u32)__popc(peers & lt)] = kv;
                    }
                }
            }
        }
    }
    if (!SCATTER) {
        err = __reduce_or_sync(0xFFFFFFFFu, err);
        nup = __reduce_add_sync(0xFFFFFFFFu, nup);
        ndown = __reduce_add_sync(0xFFFFFFFFu, ndown);
        nkey = __reduce_add_sync(0xFFFFFFFFu, nkey);
        if (lane == 0) {
            if (err) atomicOr(&ctr->verr, err);
            if (nup) atomicAdd(cnt, (unsigned long long)nup);
            if (ndown) atomicAdd(cnt + 1, (unsigned long long)ndown);
            if (nkey) atomicAdd(cnt + 2, (unsigned long long)nkey);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < VAL_BINS; i += WCH_BLOCK) hist[(i64)i * gridDim.x + blockIdx.x] = s_bin[i];
    }
}

struct ValHistLoad {
    const u32* h;
    __device__ __forceinline__ u32 operator()(i64 i) const { return h[i]; }
};
struct ValBaseStore {
    u32* b;
    __device__ __forceinline__ void operator()(i64 i, u32 ex, u32) const { b[i] = ex; }
};

__device__ __forceinline__ void val_check_key(const i64* __restrict__ off, const int32_t* __restrict__ tgt, u64 kv,
                                              Ctr* ctr) {
    const int32_t u = (int32_t)(u32)kv, w = (int32_t)((u32)(kv >> 32) & 0x7FFFFFFFu);
    const i64 ws = off[w], we = off[(i64)w + 1];
    const i64 q = lower_bound_row(tgt, ws, we, u);
    i64 c = 1;
    if (kv & VAL_DUP) {
        const i64 rs = off[u], re = off[(i64)u + 1];
        i64 p = lower_bound_row(tgt, rs, re, w);
        c = 0;
        while (p + c < re && tgt[p + c] == w) ++c;
    }
    bool bad = q + c > we || (q + c < we && tgt[q + c] == u);
    for (i64 j = 0; j < c && !bad; ++j) bad = tgt[q + j] != u;
    if (bad) atomicOr(&ctr->verr, VERR_NOTSYM);
}

static inline unsigned val_grid(i64 m) {
    unsigned b = chunk_blocks(m);
    return b < (unsigned)VAL_GRID ? b : (unsigned)VAL_GRID;
}


// One key per thread (grid-stride; the key count is read on the device, so the check can
// be queued without a host round trip): row w must hold exactly c copies of u (c = 1
// unless the key is flagged, then c is re-counted in row u).  Runs only when the counts
// balance (cnt[0] == cnt[1]); otherwise the streaming half already failed.
__global__ void k_val_check(const i64* __restrict__ off, const int32_t* __restrict__ tgt, const u64* __restrict__ keys,
                            const unsigned long long* __restrict__ cnt, Ctr* ctr) {
    if (cnt[0] != cnt[1]) return;
    const i64 nkeys = (i64)cnt[2];
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < nkeys; i += (i64)gridDim.x * blockDim.x)
        val_check_key(off, tgt, keys[i], ctr);
}

struct ValWs {
    Ctr* ctr;
    unsigned long long* cnt;   // up, down, keys
    u32 *CROW, *HIST, *BASE;
    u64 *SCAN, *KEYS;
};

static size_t carve_val(ValWs& v, char* base, i64 n, i64 m) {
    size_t o = 0;
    auto take = [&](size_t bytes) -> char* {
        o = (o + 255) & ~(size_t)255;
        char* p = base ? base + o : nullptr;
        o += bytes;
        return p;
    };
    (void)n;
    const i64 nh = (i64)VAL_BINS * val_grid(m);
    v.ctr = (Ctr*)take(sizeof(Ctr));
    v.cnt = (unsigned long long*)take(4 * sizeof(unsigned long long));
    v.CROW = (u32*)take(4 * (num_chunks(m) + 1));
    v.HIST = (u32*)take(4 * nh);
    v.BASE = (u32*)take(4 * nh);
    v.SCAN = (u64*)take(scan_status_bytes(nh));
    v.KEYS = (u64*)take(8 * (size_t)(m / 2 > 0 ? m / 2 : 1));   // keys <= #up == #down <= m/2
    return o + 256;
}

// --------------------------------------------------------------------------
// host orchestration
// --------------------------------------------------------------------------
static inline unsigned nblk(i64 items, int bs) { return (unsigned)(items > 0 ? cdiv(items, bs) : 1); }

// First-CC knobs for sweeps: PASGAL_BCC_CC=vgc|afforest forces a path (k_cc_policy
// decides otherwise), PASGAL_BCC_VGC_TAU sets tau.
static int cc_mode() {
    const char* e = getenv("PASGAL_BCC_CC");
    return e && e[0] == 'v' ? 1 : e && e[0] == 'a' ? 2 : 0;
}
static int vgc_tau() {
    const char* t = getenv("PASGAL_BCC_VGC_TAU");
    return t && atoi(t) > 0 ? atoi(t) : VGC_TAU_DEFAULT;
}
// Leaf trimming of the Euler tour (S3) pays where the spanning forest is leafy and large: the
// sampled union-find forest of a graph with >= 4 slots per vertex (RMAT, kNN: most vertices
// hook onto a neighbour and nothing hooks onto them; C5a rooting 31.8 -> 27.5 ms, C4 -1.2 ms),
// not on a lattice (C3: +0.8 ms) nor on small graphs.  PASGAL_BCC_TRIM=0/1 forces it (A/B sweeps).  Tour positions must
// stay below the HAB tags (n < 2^31 - 2).
static bool leaf_trim(i64 n, i64 m) {
    const char* e = getenv("PASGAL_BCC_TRIM");
    if (n < 64 || n >= ((i64)1 << 31) - 2) return false;
    if (e) return e[0] != '0';
    return m >= 4 * n && n >= ((i64)1 << 22);   // below 2^22 (C2: 1.21 -> 1.35 ms) the fixed costs win
}

// The direction bits (M/8 bytes) live in the dead Euler-tour array T (16 bytes per vertex).
static bool dir_bits(i64 n, i64 m) {
    const char* e = getenv("PASGAL_BCC_DIR");
    if (e && e[0] == '0') return false;
    return (u64)cdiv(m, WCH) * WCH / 8 <= (u64)16 * (u64)(n > 0 ? n : 1);
}

// Two-level tags (code table + exact gathers of the extreme slots only): PASGAL_BCC_TAGS2=0/1
// forces it.
static bool tags_two_level(i64 n, i64 m, const int32_t* tgt) {
    const char* e = getenv("PASGAL_BCC_TAGS2");
    (void)tgt;
    if (m < 1) return false;
    if (e) return e[0] != '0';
    // Its cost per slot does not depend on n (the code table stays in L2), k_tags_blk's grows
    // with FIRST / L2: RMAT 2^26 5.7 vs 7.2 ms, 2^28 35.5 vs 27.8 ms.  Short rows (kNN, grids)
    // gather two exact values per row anyway: C4 3.6 vs 4.9 ms.
    // "from 2^27 vertices" on a B200: FIRST (4 bytes per vertex) at least 4x the L2
    static i64 l2 = 0;
    if (!l2) {
        int dev = 0, bytes = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&bytes, cudaDevAttrL2CacheSize, dev) != cudaSuccess || bytes <= 0)
            bytes = 126 << 20;
        l2 = bytes;
    }
    return n >= l2 && m >= 8 * n;
}

static unsigned vgc_grid() {
    static int blocks = 0;
    if (!blocks) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_vgc_search, VGC_WARPS * 32, 0) != cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        blocks = per_sm * sms;
    }
    return (unsigned)blocks;
}

// Per-function attributes (idempotent; set outside any stream capture).
#ifndef PG_TAGS_CARVE
#define PG_TAGS_CARVE 25
#endif
static cudaError_t set_kernel_attributes() {
    cudaError_t e = cudaSuccess;
    auto chk = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
    // The list-ranking walks hit L1 (the tour revisits nearby arcs), so they ask for the
    // smallest shared-memory carveout that fits them (C5a listrank 11.85 -> 11.6 ms).
    chk(cudaFuncSetAttribute(k_lr_walk1, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    chk(cudaFuncSetAttribute(k_lr_walk2, cudaFuncAttributePreferredSharedMemoryCarveout, 30));
    // k_tags_blk likewise: its FIRST gathers need L1 lines while in flight, and a larger
    // carveout than the 6 x 8.5 KB it needs cost up to 2.5x (C5a tags 36.2 -> 34.6 ms at 25 %,
    // 90.7 ms at 100 %)
    if (PG_TAGS_CARVE >= 0)
        chk(cudaFuncSetAttribute(k_tags_blk<true>, cudaFuncAttributePreferredSharedMemoryCarveout, PG_TAGS_CARVE));
#ifdef PG_TAGS2_CARVE
    chk(cudaFuncSetAttribute(k_tags2_blk, cudaFuncAttributePreferredSharedMemoryCarveout, PG_TAGS2_CARVE));
#endif
    chk(cudaFuncSetAttribute(k_wyllie_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(2 * sizeof(u32) * WY_MAX)));
    (void)vgc_grid();   // occupancy query cached outside any capture
    return e;
}

int bcc_launch(const pasgal_csr_t* g, const pasgal_bcc_out_t* out, void* ws_ptr, size_t ws_bytes, u64 seed,
               u32 flags, cudaStream_t st, pasgal_bcc_prof_t* prof) {
    const i64 n = g->n, m = g->m_slots;
    const i64 L = 2 * n;
    Ws w;
    size_t need = carve(w, nullptr, n, m);
    if (ws_bytes < need) return PASGAL_EWORKSPACE;
    carve(w, (char*)ws_ptr, n, m);
    const i64* off = g->offsets;
    const int32_t* tgt = g->targets;
    const int B = 256;
    int nl = 0;  // kernel launches issued by this call
    // stage boundaries: the caller's CUDA events, and NVTX ranges named after the stages
    // (host launch intervals in nsys / ncu --nvtx; no cost without an attached tool)
    static const char* const stage_names[PASGAL_BCC_NSTAGES] = {
        "pasgal_bcc", "first_cc", "forest", "listrank", "tour", "tags", "rmq", "last_cc", "artic", "labels",
        "canonical"};
    int nvtx_open = 0;
    auto mark = [&](int stage) -> cudaError_t {
        if (nvtx_open) {
            nvtxRangePop();
            nvtx_open = 0;
        }
        if (stage + 1 < PASGAL_BCC_NSTAGES) {
            nvtxRangePushA(stage_names[stage + 1]);
            nvtx_open = 1;
        }
        if (prof && prof->events && stage < prof->n_events && prof->events[stage])
            return cudaEventRecord((cudaEvent_t)prof->events[stage], st);
        return cudaSuccess;
    };
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    PG_CUDA_TRY(cudaStreamIsCapturing(st, &cap));
    const bool capturing = cap != cudaStreamCaptureStatusNone;
    static const bool debug_env = getenv("PASGAL_BCC_DEBUG") != nullptr;
    const bool debug = debug_env && !capturing;
#define PG_K(...)                                                                          \
    do {                                                                                   \
        __VA_ARGS__;                                                                       \
        ++nl;                                                                              \
        if (debug) {                                                                       \
            cudaError_t e_ = cudaStreamSynchronize(st);                                    \
            if (e_ == cudaSuccess) e_ = cudaGetLastError();                                \
            if (e_ != cudaSuccess) {                                                       \
                fprintf(stderr, "pasgal_bcc: launch %d (%s) failed: %s\n", nl, #__VA_ARGS__, \
                        cudaGetErrorString(e_));                                           \
                return PASGAL_ECUDA;                                                       \
            }                                                                              \
        }                                                                                  \
    } while (0)

    if (!capturing) PG_CUDA_TRY(set_kernel_attributes());
    PG_CUDA_TRY(mark(PASGAL_STAGE_BEGIN));
    PG_CUDA_TRY(cudaMemsetAsync(w.ctr, 0, sizeof(Ctr), st));
    PG_CUDA_TRY(cudaMemsetAsync(out->artic_bits, 0, sizeof(u32) * (size_t)cdiv(n, 32), st));
    if (n == 0) {
        PG_K(k_finish<<<1, 1, 0, st>>>(w.ctr, out->bcc_count));
        PG_LAUNCH_CHECK();
        for (int s = PASGAL_STAGE_BEGIN + 1; s < PASGAL_BCC_NSTAGES; ++s) PG_CUDA_TRY(mark(s));
        if (prof) prof->launches = nl;
        return PASGAL_OK;
    }
    // ---- S2 First-CC: VGC local searches on sparse local-id graphs, sampled union-find
    // otherwise (k_cc_policy decides on the device; the other path's kernels return at once)
    const int lb = local_lb(n);
    // VGC is a candidate only for sparse graphs (host-known sizes); then k_cc_policy picks
    // on the device and the other path's kernels return at once.  k_vgc_init runs
    // grid-stride on a capped grid; k_cc_sample / k_cc_rest keep one vertex per thread of a
    // full grid (a capped grid-stride or chunked form let the in-flight vertices spread over
    // the id range: C4 k_cc_sample 3.0 -> 8.3 ms), which costs ~0.1 ms when skipped (C3)
    const int mode = cc_mode();
    const bool vgc_possible = mode == 1 || (mode == 0 && n >= VGC_MIN_N && m <= VGC_MAX_DEG * n);
    const u32* gate = vgc_possible ? &w.ctr->cc_vgc : nullptr;
    // leaf trimming (section S3 below) places no out-arc at hook time: the arcs of a leaf's
    // edge never enter a list
    const bool trim = leaf_trim(n, m);
    const HookRec hook{w.HAB, trim ? nullptr : w.HEAD, w.NEXT};
    const unsigned capped = (unsigned)(nblk(n, B) < 148 * 8 ? nblk(n, B) : 148 * 8);
    if (vgc_possible) {
        PG_K(k_cc_policy<<<1, POLICY_SAMPLES, 0, st>>>(n, m, off, tgt, seed, mode, w.ctr));
        PG_K(k_vgc_init<<<capped, B, 0, st>>>(n, off, w.P, w.HAB, w.HEAD, w.CROW, gate));
        PG_K(k_vgc_search<<<vgc_grid(), VGC_WARPS * 32, 0, st>>>(n, off, tgt, w.P, hook, w.UOFF, w.ctr, vgc_tau(),
                                                                 gate));
        PG_K(k_vgc_rest<<<148 * 8, B, 0, st>>>(n, off, tgt, w.P, hook, w.UOFF, w.ctr, w.HEAVY, gate));
        PG_K(k_cc_rest_heavy<0><<<HEAVY_GRID, 256, 0, st>>>(n, off, tgt, w.P, hook, w.ctr, w.HEAVY, gate, 1));
    }
    PG_K(k_cc_local<<<(unsigned)cdiv(n, (i64)1 << lb), LOCAL_T, 0, st>>>(n, lb, off, tgt, w.P, w.HAB, w.HEAD,
                                                                         trim ? nullptr : w.NEXT, w.CROW, gate));
    PG_K(k_cc_sample<<<nblk(n, B), B, 0, st>>>(n, lb, off, tgt, w.P, hook, gate));
    PG_K(k_compress<COMPRESS_ILP><<<nblk(cdiv(n, COMPRESS_ILP), B), B, 0, st>>>(n, w.P, gate));
    PG_K(k_giant<<<1, GIANT_SAMPLES, 0, st>>>(n, w.P, seed, &w.ctr->giant, gate));
    PG_K(k_cc_rest<<<nblk(n, B), B, 0, st>>>(n, off, tgt, w.P, hook, w.ctr, w.HEAVY, gate));
    PG_K(k_cc_rest_heavy<NSAMPLE><<<HEAVY_GRID, 256, 0, st>>>(n, off, tgt, w.P, hook, w.ctr, w.HEAVY, gate, 0));
    // no final compress: later stages only ask "is x a root", and P[x] == x exactly at roots
    PG_LAUNCH_CHECK();
    PG_CUDA_TRY(mark(PASGAL_STAGE_FIRST_CC));
    // ---- S3 rooting: arc lists
    // forest marks: ONE in GBIT (free until Last-CC), TWO and ROOT inside UCNT (free until
    // canonicalisation); leaves per parent in UOFF (free after First-CC)
    ForestMarks fm{nullptr, nullptr, nullptr, nullptr};
    u32* LCNT = trim ? w.UOFF : nullptr;
    if (trim) {
        const i64 nw = cdiv(n, 32);
        fm = ForestMarks{w.GBIT, w.UCNT, w.UCNT + nw, w.UCNT};   // LEAF over TWO
        PG_CUDA_TRY(cudaMemsetAsync(fm.ONE, 0, 4 * (size_t)nw, st));
        PG_CUDA_TRY(cudaMemsetAsync(fm.TWO, 0, 4 * (size_t)nw, st));
        PG_CUDA_TRY(cudaMemsetAsync(LCNT, 0, 4 * (size_t)n, st));
        PG_K(k_forest_marks<<<nblk(n, B), B, 0, st>>>(n, w.HAB, fm));
    }
    if (trim) PG_K(k_leaf_bits<<<nblk(cdiv(n, 32), B), B, 0, st>>>(cdiv(n, 32), fm));
    PG_K(k_arc_link_blk<<<nblk(n, AL_T), AL_T, 0, st>>>(n, w.HAB, w.HEAD, w.NEXT, !trim, fm, LCNT, w.PM, w.ctr));
    PG_K(k_arc_close<<<nblk(n, AC_B * AC_V), AC_B, 0, st>>>(
        n, w.HAB, w.HEAD, w.P, fm, w.ctr, w.NEXT,
        IsoOut{w.FL, w.ROOTMARK}));
    PG_LAUNCH_CHECK();
    PG_CUDA_TRY(mark(PASGAL_STAGE_FOREST));
    // ---- S3 list ranking
    PG_K(k_lr_walk1<<<nblk(w.ns, 128), 128, 0, st>>>(n, w.ns, w.lrs, w.NEXT, w.HAB, w.HEAD, fm.ONE, w.ctr,
                                                     w.SPLEN[0], w.SPNEXT[0]));
    int cur = 0;
    if (w.ns <= WY_MAX) {
        const size_t smem = 2 * sizeof(u32) * WY_MAX;
        PG_K(k_wyllie_small<<<1, WY_T, smem, st>>>(w.ns, w.SPLEN[0], w.SPNEXT[0], w.SPLEN[1]));
        cur = 1;
    } else {
        for (i64 span = 1; span < w.ns; span <<= 1) {
            PG_K(k_wyllie<<<nblk(w.ns, B), B, 0, st>>>(w.ns, w.SPLEN[cur], w.SPNEXT[cur], w.SPLEN[cur ^ 1],
                                                       w.SPNEXT[cur ^ 1]));
            cur ^= 1;
        }
    }
    PG_K(k_lr_walk2<<<nblk(w.ns, 128), 128, 0, st>>>(n, w.ns, w.lrs, w.NEXT, w.HAB, w.HEAD, fm.ONE, w.ctr,
                                                     w.SPLEN[cur], w.HAB, w.TA));
    PG_LAUNCH_CHECK();
    PG_CUDA_TRY(mark(PASGAL_STAGE_LISTRANK));
    PG_CUDA_TRY(launch_scan<u32>(L, w.SCAN, 0u, SumOp(), PreLoad{w.TA, w.HAB, w.T, w.TP, w.ctr, n, LCNT},
                                 PreStore{w.T, w.TP, w.ctr, w.FL, w.PV, w.E, w.PPAR, w.W, trim ? w.TA : nullptr, n},
                                 (u32*)nullptr, st));
    ++nl;
    if (trim) {   // the weighted prefix (in TA) -> first/last of the tour vertices, then the leaves
        PG_K(k_pre_place<<<nblk(L, B), B, 0, st>>>(n, w.T, w.TP, w.TA, w.ctr, LCNT, w.FL, w.PV, w.E, w.PPAR, w.W,
                                                    w.HEAVY));
        PG_K(k_leaf_runs<<<HEAVY_GRID, 256, 0, st>>>(w.ctr, w.HEAVY, LCNT, w.FL, w.E, w.PPAR, w.W));
    }
    PG_K(k_vertex_first<<<nblk(n, B), B, 0, st>>>(n, w.FL, w.PPAR, w.FIRST, out->parent, out->first,
                                                   trim ? fm.LEAF : nullptr, w.PM, w.PV, w.ctr));
    PG_LAUNCH_CHECK();
    PG_CUDA_TRY(mark(PASGAL_STAGE_TOUR));
    // ---- S4 tags + RMQ (+ S5 tree-edge unions)
    // per-slot direction bits for the labels pass (first[target] > first[row]), M/8 bytes in
    // the Euler-tour array T (dead after the tour stage; room for up to 128 slots per vertex)
    u32* dir = out->edge_label && dir_bits(n, m) ? (u32*)w.T : nullptr;
    if (w.nch > 0) {
        if (tags_two_level(n, m, tgt)) {
            u32* bnd = w.TQ;
            u32* Q = w.TQ + 256;
            PG_K(k_tag_bounds<<<1, 1024, 0, st>>>(m, tgt, w.FIRST, bnd));
            PG_K(k_tag_codes<<<nblk(cdiv(n, (i64)1 << TAG_PW_SH), 256), 256, 0, st>>>(n, w.FIRST, bnd, Q));
            PG_K(k_tags2_blk<<<chunk_blocks(m), WCH_BLOCK, 0, st>>>(off, tgt, n, m, w.CROW, w.FIRST, Q, w.W, dir));
        } else if (n >= ((i64)1 << 22))
            PG_K(k_tags_blk<true><<<chunk_blocks(m), WCH_BLOCK, 0, st>>>(off, tgt, n, m, w.CROW, w.FIRST, w.W, dir));
        else
            PG_K(k_tags_blk<false><<<chunk_blocks(m), WCH_BLOCK, 0, st>>>(off, tgt, n, m, w.CROW, w.FIRST, w.W, dir));
    }
    PG_LAUNCH_CHECK();
    PG_CUDA_TRY(mark(PASGAL_STAGE_TAGS));
    PG_K(k_rmq_block<<<nblk(n, B), B, 0, st>>>(n, w.W, w.PM, w.ST, w.ctr));
    if (w.nb <= RMQ_SMALL) {
        if (w.lv > 1) PG_K(k_rmq_levels_small<<<1, 1024, 0, st>>>(w.nb, w.lv, w.ST));
    } else {
        for (i64 k = 1; k < w.lv; ++k)
            PG_K(k_rmq_level<<<nblk(w.nb, B), B, 0, st>>>(w.nb, w.ST + (k - 1) * w.nb, w.ST + k * w.nb,
                                                          (i64)1 << (k - 1), w.ctr));
    }
    PG_K(k_rmq_query<<<nblk(n, B), B, 0, st>>>(n, w.W, w.E, w.PV, w.PPAR, w.PM, w.ST, w.nb, w.FL, w.FPF, w.ctr));
    PG_LAUNCH_CHECK();
    PG_CUDA_TRY(mark(PASGAL_STAGE_RMQ));
    // ---- S5 Last-CC over cross edges
    PG_K(k_cc2_local<<<(unsigned)cdiv(n, (i64)1 << lb), LOCAL_T, 0, st>>>(n, lb, w.FPF, w.W, w.E, w.C, w.ctr));
    PG_K(k_cc2_links<<<nblk(n, B), B, 0, st>>>(n, lb, w.FPF, w.W, w.E, w.C, w.ctr));
    PG_K(k_compress<COMPRESS_ILP2><<<nblk(cdiv(n, COMPRESS_ILP2), B), B, 0, st>>>(n, w.C, nullptr, &w.ctr->niso));
    PG_K(k_giant<<<1, GIANT_SAMPLES, 0, st>>>(n, w.C, seed + 0x9E3779B97F4A7C15ull, &w.ctr->giant2, nullptr));
    PG_K(k_cc2_rest<<<nblk(n, B), B, 0, st>>>(n, off, tgt, w.FL, w.PV, w.E, w.P, w.C, w.ctr, w.HEAVY));
    PG_K(k_cc2_rest_heavy<<<HEAVY_GRID, 256, 0, st>>>(n, off, tgt, w.FL, w.C, w.ctr, w.HEAVY));
    PG_K(k_compress_final<<<nblk(cdiv(n, COMPRESS_ILP2), B), B, 0, st>>>(n, w.C, w.ctr));
    PG_K(k_cid_vertices<<<nblk(n, B), B, 0, st>>>(n, w.C, w.FIRST, w.ctr, w.CIDV, w.GBIT, out->comp));
    PG_LAUNCH_CHECK();
    PG_CUDA_TRY(mark(PASGAL_STAGE_LAST_CC));
    // ---- S6 articulation, labels, count
    PG_K(k_artic<<<nblk(n, B), B, 0, st>>>(n, w.PPAR, w.FPF, w.C, w.P, w.ROOTMARK, out->artic_bits, w.ctr));
    PG_LAUNCH_CHECK();
    PG_CUDA_TRY(mark(PASGAL_STAGE_ARTIC));
    if (w.nch > 0 && out->edge_label)
        PG_K(k_labels<<<chunk_blocks(m), WCH_BLOCK, 0, st>>>(off, tgt, n, m, w.CROW, w.CIDV, w.GBIT, w.ctr, dir,
                                                             out->edge_label));
    PG_K(k_finish<<<1, 1, 0, st>>>(w.ctr, out->bcc_count));
    PG_LAUNCH_CHECK();
    PG_CUDA_TRY(mark(PASGAL_STAGE_LABELS));
    if (flags & PASGAL_BCC_CANONICAL) {
        PG_K(k_canon_init<<<nblk(n, B), B, 0, st>>>(n, w.UCNT, n, w.CANON));
        if (w.nch > 0) PG_K(k_canon_count<<<chunk_blocks(m), WCH_BLOCK, 0, st>>>(off, tgt, n, m, w.CROW, w.UCNT));
        PG_CUDA_TRY(launch_scan<u32>(n, w.SCAN, 0u, SumOp(), UcntLoad{w.UCNT}, UoffStore{w.UOFF}, (u32*)nullptr, st));
        ++nl;
        if (w.nch > 0)
            PG_K(k_canon_min<<<chunk_blocks(m), WCH_BLOCK, 0, st>>>(off, tgt, n, m, w.CROW, w.UCNT, w.UOFF,
                                                                   out->edge_label, n, w.CANON));
        if (m > 0) PG_K(k_canon_apply<<<nblk(m, B), B, 0, st>>>(m, w.CANON, n, out->edge_label, out->edge_label));
        PG_LAUNCH_CHECK();
    }
    PG_CUDA_TRY(mark(PASGAL_STAGE_CANONICAL));
#undef PG_K
    if (prof) prof->launches = nl;
    return PASGAL_OK;
}

// ----------------------------------------------------------------------------
// CUDA-graph form of one pasgal_bcc call: the ~50-70 launches of a call captured once for
// fixed pointers and sizes, then replayed with one launch (small graphs are launch-bound:
// C1 is ~0.5 ms of mostly launch gaps).  Kernels read every data-dependent count from the
// workspace, so a replay is exactly a fresh call on whatever the pointers hold.
// ----------------------------------------------------------------------------
struct BccGraph {
    cudaGraphExec_t exec;
    int launches;
};

int bcc_graph_create(const pasgal_csr_t* g, const pasgal_bcc_out_t* out, void* ws, size_t ws_bytes, u64 seed,
                     u32 flags, void** handle) {
    *handle = nullptr;
    PG_CUDA_TRY(set_kernel_attributes());
    cudaStream_t cs;
    PG_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    pasgal_bcc_prof_t prof{nullptr, 0, 0};
    int st = PASGAL_OK;
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        st = bcc_launch(g, out, ws, ws_bytes, seed, flags, cs, &prof);
        e = cudaStreamEndCapture(cs, &graph);
    }
    cudaStreamDestroy(cs);
    if (st != PASGAL_OK || e != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        return st != PASGAL_OK ? st : PASGAL_ECUDA;
    }
    cudaGraphExec_t exec;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return PASGAL_ECUDA;
    *handle = new BccGraph{exec, prof.launches};
    return PASGAL_OK;
}

int bcc_graph_launch(void* handle, cudaStream_t st, int* launches) {
    BccGraph* h = (BccGraph*)handle;
    PG_CUDA_TRY(cudaGraphLaunch(h->exec, st));
    if (launches) *launches = h->launches;
    return PASGAL_OK;
}

void bcc_graph_destroy(void* handle) {
    BccGraph* h = (BccGraph*)handle;
    if (!h) return;
    cudaGraphExecDestroy(h->exec);
    delete h;
}

// ----------------------------------------------------------------------------
// stand-alone connected components: S2 alone.  Union by
// index makes every component's root its minimum vertex id, so the output is deterministic
// and equal to a sequential labelling by minimum id.
// ----------------------------------------------------------------------------
__global__ void k_cc_out(i64 n, const u32* __restrict__ P, u32* comp, Ctr* ctr) {
    i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    u32 isroot = 0;
    if (v < n) {
        u32 r = P[v];
        comp[v] = r;
        isroot = r == (u32)v;
    }
    u32 cnt = __popc(__ballot_sync(0xFFFFFFFFu, isroot));
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&ctr->ncomp, cnt);
}

__global__ void k_cc_count(const Ctr* ctr, i64* count) { *count = ctr->ncomp; }

int cc_launch(const pasgal_csr_t* g, uint32_t* comp, int64_t* count_dev, void* ws_ptr, size_t ws_bytes, u64 seed,
              cudaStream_t st) {
    const i64 n = g->n;
    Ws w;
    size_t need = carve(w, nullptr, n, g->m_slots);
    if (ws_bytes < need) return PASGAL_EWORKSPACE;
    carve(w, (char*)ws_ptr, n, g->m_slots);
    const i64* off = g->offsets;
    const int32_t* tgt = g->targets;
    const int B = 256;
    PG_CUDA_TRY(cudaMemsetAsync(w.ctr, 0, sizeof(Ctr), st));
    if (n > 0) {
        const int lb = local_lb(n);
        const HookRec rec{w.HAB, nullptr, nullptr};   // forest edges only: no out-arc lists here
        k_cc_local<<<(unsigned)cdiv(n, (i64)1 << lb), LOCAL_T, 0, st>>>(n, lb, off, tgt, w.P, w.HAB, w.HEAD, nullptr,
                                                                        nullptr, nullptr);
        k_cc_sample<<<nblk(n, B), B, 0, st>>>(n, lb, off, tgt, w.P, rec, nullptr);
        k_compress<COMPRESS_ILP><<<nblk(cdiv(n, COMPRESS_ILP), B), B, 0, st>>>(n, w.P, nullptr);
        k_giant<<<1, GIANT_SAMPLES, 0, st>>>(n, w.P, seed, &w.ctr->giant, nullptr);
        k_cc_rest<<<nblk(n, B), B, 0, st>>>(n, off, tgt, w.P, rec, w.ctr, w.HEAVY, nullptr);
        k_cc_rest_heavy<NSAMPLE><<<HEAVY_GRID, 256, 0, st>>>(n, off, tgt, w.P, rec, w.ctr, w.HEAVY, nullptr, 0);
        k_compress<COMPRESS_ILP><<<nblk(cdiv(n, COMPRESS_ILP), B), B, 0, st>>>(n, w.P, nullptr);
        k_cc_out<<<nblk(n, B), B, 0, st>>>(n, w.P, comp, w.ctr);
    }
    k_cc_count<<<1, 1, 0, st>>>(w.ctr, count_dev);
    PG_LAUNCH_CHECK();
    return PASGAL_OK;
}

// ----------------------------------------------------------------------------
// stand-alone canonicaliser (results.py:91-112): any per-slot labelling
// with ids in [0, nlab) -> every slot labelled by the minimum undirected edge id of its
// class.  Ids outside [0, nlab) (e.g. 0xFFFFFFFF = unlabelled) pass through unchanged.
// ----------------------------------------------------------------------------
struct CanonWs {
    u32 *UCNT, *UOFF, *CANON, *CROW;
    u64* SCAN;
};
static size_t canon_carve(CanonWs& c, char* base, i64 n, i64 m, i64 nlab) {
    size_t o = 0;
    auto take = [&](size_t bytes) -> char* {
        o = (o + 255) & ~(size_t)255;
        char* p = base ? base + o : nullptr;
        o += bytes;
        return p;
    };
    i64 nn = n > 0 ? n : 1;
    c.UCNT = (u32*)take(4 * nn);
    c.UOFF = (u32*)take(4 * nn);
    c.CANON = (u32*)take(4 * (nlab > 0 ? nlab : 1));
    c.CROW = (u32*)take(4 * (num_chunks(m) + 1));
    c.SCAN = (u64*)take(scan_status_bytes(nn));
    return o + 256;
}

size_t canonicalize_temp_bytes(i64 n, i64 m, i64 nlab) {
    CanonWs c;
    return canon_carve(c, nullptr, n, m, nlab);
}

int canonicalize_launch(const pasgal_csr_t* g, const u32* in, i64 nlab, u32* out, void* temp, size_t temp_bytes,
                        cudaStream_t st) {
    const i64 n = g->n, m = g->m_slots;
    CanonWs c;
    if (temp_bytes < canon_carve(c, nullptr, n, m, nlab)) return PASGAL_EWORKSPACE;
    canon_carve(c, (char*)temp, n, m, nlab);
    const int B = 256;
    const i64 nch = num_chunks(m);
    const i64* off = g->offsets;
    const int32_t* tgt = g->targets;
    if (n == 0 || m == 0) return PASGAL_OK;
    i64 init = n > nlab ? n : nlab;
    k_canon_init<<<nblk(init, B), B, 0, st>>>(n, c.UCNT, nlab, c.CANON);
    k_chunk_rows<<<nblk(nch, B), B, 0, st>>>(off, n, m, nch, c.CROW);
    k_canon_count<<<chunk_blocks(m), WCH_BLOCK, 0, st>>>(off, tgt, n, m, c.CROW, c.UCNT);
    PG_CUDA_TRY(launch_scan<u32>(n, c.SCAN, 0u, SumOp(), UcntLoad{c.UCNT}, UoffStore{c.UOFF}, (u32*)nullptr, st));
    k_canon_min<<<chunk_blocks(m), WCH_BLOCK, 0, st>>>(off, tgt, n, m, c.CROW, c.UCNT, c.UOFF, in, nlab, c.CANON);
    k_canon_apply<<<nblk(m, B), B, 0, st>>>(m, c.CANON, nlab, in, out);
    PG_LAUNCH_CHECK();
    return PASGAL_OK;
}

// first offending index of a CSR for positioned load errors (graph.py:380-395 semantics):
// out[0] = first i with off[i] > off[i+1], out[1] = first slot with a target outside [0,n)
__global__ void k_first_bad_offset(i64 n, const i64* __restrict__ off, unsigned long long* out) {
    i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && off[i] > off[i + 1]) atomicMin(out, (unsigned long long)(i + 1));
}
__global__ void k_first_bad_target(i64 n, i64 m, const int32_t* __restrict__ tgt, unsigned long long* out) {
    i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < m && (tgt[s] < 0 || (i64)tgt[s] >= n)) atomicMin(out + 1, (unsigned long long)s);
}
int csr_first_error(const pasgal_csr_t* g, void* scratch, int64_t* host_out, cudaStream_t st) {
    const i64 n = g->n, m = g->m_slots;
    unsigned long long* d = (unsigned long long*)scratch;
    PG_CUDA_TRY(cudaMemsetAsync(d, 0xFF, 2 * sizeof(unsigned long long), st));
    const int B = 256;
    if (n > 0) k_first_bad_offset<<<nblk(n, B), B, 0, st>>>(n, g->offsets, d);
    if (m > 0) k_first_bad_target<<<nblk(m, B), B, 0, st>>>(n, m, g->targets, d);
    unsigned long long h[2];
    PG_CUDA_TRY(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, st));
    PG_CUDA_TRY(cudaStreamSynchronize(st));
    host_out[0] = h[0] == ~0ull ? -1 : (int64_t)h[0];
    host_out[1] = h[1] == ~0ull ? -1 : (int64_t)h[1];
    return PASGAL_OK;
}

bool bcc_two_level_tags(i64 n, i64 m) { return tags_two_level(n, m, nullptr); }

size_t bcc_workspace_bytes(i64 n, i64 m) {
    Ws w;
    return carve(w, nullptr, n, m);
}

size_t validate_workspace_bytes(i64 n, i64 m) {
    ValWs v;
    return carve_val(v, nullptr, n, m);
}

// bitmap word k -> bytes [32k, 32k+32) (0/1), two 16-byte stores per thread; the tail word
// writes only its n - 32k valid bytes.
__global__ void k_bits_to_bytes(const u32* __restrict__ bits, i64 n, uint8_t* __restrict__ out) {
    const i64 k = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const i64 b0 = k * 32;
    if (b0 >= n) return;
    const u32 x = bits[k];
    if (b0 + 32 <= n && ((uintptr_t)out & 15) == 0) {
        u32 wv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const u32 nib = (x >> (4 * j)) & 0xFu;
            wv[j] = (nib & 1u) | ((nib >> 1 & 1u) << 8) | ((nib >> 2 & 1u) << 16) | ((nib >> 3 & 1u) << 24);
        }
        uint4* o = reinterpret_cast<uint4*>(out + b0);
        o[0] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        o[1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
    } else {
        for (int j = 0; j < 32 && b0 + j < n; ++j) out[b0 + j] = (uint8_t)(x >> j & 1u);
    }
}

int bits_to_bytes(const u32* bits, i64 n, uint8_t* out, cudaStream_t st) {
    if (n <= 0) return PASGAL_OK;
    const i64 words = cdiv(n, 32);
    k_bits_to_bytes<<<nblk(words, 256), 256, 0, st>>>(bits, n, out);
    PG_LAUNCH_CHECK();
    return PASGAL_OK;
}

// Run checksum (results.canonical_checksum's device twin): out[0] += sum over slots of
// lab[s] * (((s * 0x9E3779B1) mod 2^32) | 1) mod 2^64 (unsigned wraparound), out[1] += the
// articulation popcount.  One grid-stride pass, a warp reduction and one atomic per warp.
__global__ void k_checksum(const u32* __restrict__ lab, i64 m, const u32* __restrict__ bits, i64 nw,
                           unsigned long long* out) {
    const i64 stride = (i64)gridDim.x * blockDim.x;
    u64 h = 0, c = 0;
    for (i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x; s < m; s += stride)
        h += (u64)__ldcs(lab + s) * (u64)((u32)((u64)s * 0x9E3779B1ull) | 1u);
    for (i64 k = (i64)blockIdx.x * blockDim.x + threadIdx.x; k < nw; k += stride) c += __popc(bits[k]);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        h += __shfl_xor_sync(0xFFFFFFFFu, h, o);
        c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (h) atomicAdd(out, (unsigned long long)h);
        if (c) atomicAdd(out + 1, (unsigned long long)c);
    }
}

int canonical_checksum(const u32* lab, i64 m, const u32* bits, i64 n, unsigned long long* out, cudaStream_t st) {
    PG_CUDA_TRY(cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), st));
    const i64 work = m > cdiv(n, 32) ? m : cdiv(n, 32);
    if (work <= 0) return PASGAL_OK;
    i64 blocks = cdiv(work, 256 * 8);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_checksum<<<(unsigned)blocks, 256, 0, st>>>(lab, m, bits, cdiv(n, 32), out);
    PG_LAUNCH_CHECK();
    return PASGAL_OK;
}

static int val_status(u32 verr) {
    if (verr & VERR_RANGE) return PASGAL_ERANGE;
    if (verr & VERR_UNSORTED) return PASGAL_EUNSORTED;
    if (verr & VERR_NOTSYM) return PASGAL_ENOTSYM;
    return PASGAL_OK;
}

static int val_shift(i64 n) {
    int bits = 0;
    while (bits < 40 && ((n - 1) >> bits) != 0) ++bits;   // bit length of n - 1
    return bits > VAL_BINS_LB ? bits - VAL_BINS_LB : 0;
}

// Small results of the streaming checks go to the host through mapped pinned memory
// written by a one-thread kernel, not cudaMemcpy: a D2H copy of a few bytes queues behind
// any large D2H on the copy engine (in BccPipeline, the previous graph's 17 GB of labels),
// which held each graph's BCC back ~185 ms at RMAT 2^28.  One buffer per host thread keeps
// the library reentrant; a call finishes with it before returning.
struct ValReadback {
    unsigned long long verr, up, down, keys;
};

__global__ void k_val_publish(const Ctr* ctr, const unsigned long long* cnt, volatile ValReadback* h) {
    h->verr = ctr->verr;
    h->up = cnt ? cnt[0] : 0ull;
    h->down = cnt ? cnt[1] : 0ull;
    h->keys = cnt ? cnt[2] : 0ull;
}

static cudaError_t val_readback(const Ctr* ctr, const unsigned long long* cnt, cudaStream_t st, ValReadback* out) {
    thread_local ValReadback* hbuf = nullptr;
    thread_local ValReadback* dbuf = nullptr;
    if (!hbuf) {
        cudaError_t e = cudaHostAlloc((void**)&hbuf, sizeof(ValReadback), cudaHostAllocMapped | cudaHostAllocPortable);
        if (e != cudaSuccess) return e;
        e = cudaHostGetDevicePointer((void**)&dbuf, hbuf, 0);
        if (e != cudaSuccess) return e;
    }
    k_val_publish<<<1, 1, 0, st>>>(ctr, cnt, dbuf);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
        const volatile ValReadback* v = hbuf;
        out->verr = v->verr;
        out->up = v->up;
        out->down = v->down;
        out->keys = v->keys;
    }
    return e;
}

// Validation, first half: the streaming checks (ranges, row order, #up == #down, and the
// bucket histogram of the keys), waited for.  After PASGAL_OK the CSR is safe for
// FAST-BCC.  A nonzero return is final.
int csr_validate_begin(const pasgal_csr_t* g, void* ws_ptr, size_t ws_bytes, cudaStream_t st) {
    const i64 n = g->n, m = g->m_slots;
    ValWs v;
    size_t need = carve_val(v, nullptr, n, m);
    if (ws_bytes < need) return PASGAL_EWORKSPACE;
    carve_val(v, (char*)ws_ptr, n, m);
    PG_CUDA_TRY(cudaMemsetAsync(v.ctr, 0, sizeof(Ctr), st));
    PG_CUDA_TRY(cudaMemsetAsync(v.cnt, 0, 4 * sizeof(unsigned long long), st));
    const int B = 256;
    k_validate_offsets<<<nblk(n + 1, B), B, 0, st>>>(n, m, g->offsets, v.ctr);
    PG_LAUNCH_CHECK();
    ValReadback h;
    PG_CUDA_TRY(val_readback(v.ctr, nullptr, st, &h));
    if (h.verr & VERR_RANGE) return PASGAL_ERANGE;
    if (m == 0 || n == 0) return PASGAL_OK;
    const i64 nch = num_chunks(m);
    const unsigned grid = val_grid(m);
    k_chunk_rows<<<nblk(nch, B), B, 0, st>>>(g->offsets, n, m, nch, v.CROW);
    k_val_pass<false><<<grid, WCH_BLOCK, 0, st>>>(g->offsets, g->targets, n, m, v.CROW, val_shift(n), v.ctr, v.cnt,
                                                   v.HIST, nullptr, nullptr);
    PG_LAUNCH_CHECK();
    PG_CUDA_TRY(val_readback(v.ctr, v.cnt, st, &h));
    if (h.verr) return val_status((u32)h.verr);
    if (h.up != h.down) return PASGAL_ENOTSYM;
    return PASGAL_OK;
}

__global__ void k_val_status(const Ctr* ctr, int32_t* status) {
    const u32 e = ctr->verr;
    *status = (e & VERR_RANGE) ? PASGAL_ERANGE : (e & VERR_UNSORTED) ? PASGAL_EUNSORTED
            : (e & VERR_NOTSYM) ? PASGAL_ENOTSYM : PASGAL_OK;
}

// Validation, second half, asynchronous: the bucketed symmetry check (scan, key scatter,
// check) is queued on `st` and its final status written to *status (device int32).  No
// host synchronisation, so the caller can order it after other work (FAST-BCC) with an
// event and let it run while the labels are copied out.
int csr_validate_check(const pasgal_csr_t* g, void* ws_ptr, size_t ws_bytes, int32_t* status, cudaStream_t st) {
    const i64 n = g->n, m = g->m_slots;
    ValWs v;
    if (ws_bytes < carve_val(v, nullptr, n, m)) return PASGAL_EWORKSPACE;
    carve_val(v, (char*)ws_ptr, n, m);
    if (m > 0 && n > 0) {
        const unsigned grid = val_grid(m);
        const i64 nh = (i64)VAL_BINS * grid;
        PG_CUDA_TRY(launch_scan<u32>(nh, v.SCAN, 0u, SumOp(), ValHistLoad{v.HIST}, ValBaseStore{v.BASE},
                                     (u32*)nullptr, st));
        k_val_pass<true><<<grid, WCH_BLOCK, 0, st>>>(g->offsets, g->targets, n, m, v.CROW, val_shift(n), v.ctr, v.cnt,
                                                      nullptr, v.BASE, v.KEYS);
        // one thread per possible key (<= m/2; the true count is read on the device): a
        // grid-stride loop over 8 CTAs per SM ran 231 ms instead of 148 at RMAT 2^28
        k_val_check<<<nblk(m / 2 > 0 ? m / 2 : 1, 256), 256, 0, st>>>(g->offsets, g->targets, v.KEYS, v.cnt, v.ctr);
        PG_LAUNCH_CHECK();
    }
    k_val_status<<<1, 1, 0, st>>>(v.ctr, status);
    PG_LAUNCH_CHECK();
    return PASGAL_OK;
}

// Validation, second half, blocking: the check above, waited for; the final status.
int csr_validate_end(const pasgal_csr_t* g, void* ws_ptr, size_t ws_bytes, cudaStream_t st) {
    ValWs v;
    if (ws_bytes < carve_val(v, nullptr, g->n, g->m_slots)) return PASGAL_EWORKSPACE;
    carve_val(v, (char*)ws_ptr, g->n, g->m_slots);
    int32_t* status = reinterpret_cast<int32_t*>(v.cnt + 3);   // spare counter word
    int s = csr_validate_check(g, ws_ptr, ws_bytes, status, st);
    if (s) return s;
    int32_t h = 0;
    PG_CUDA_TRY(cudaMemcpyAsync(&h, status, sizeof h, cudaMemcpyDeviceToHost, st));
    PG_CUDA_TRY(cudaStreamSynchronize(st));
    return h;
}

int csr_validate(const pasgal_csr_t* g, void* ws_ptr, size_t ws_bytes, cudaStream_t st) {
    int s = csr_validate_begin(g, ws_ptr, ws_bytes, st);
    return s ? s : csr_validate_end(g, ws_ptr, ws_bytes, st);
}

}  // namespace pg
