// bfs.cu -- bit-parallel multi-source BFS on the device: the searches
// behind the reference's estimate_diameter (graph.py:557-605, one FIFO BFS per sampled
// source) and its exact hop-distance BFS (oracles.bfs_queue, oracles.py:27-46).
//
// Up to 64 sources run together: every vertex carries a 64-bit SEEN mask and a FRONT mask
// (bit i = reached by source i, first time at the current level), so one pass over a
// frontier vertex's adjacency serves every source that reached it at this level.
//   k_bfs_expand  (top-down push, works on directed CSRs) one lane per frontier vertex;
//                 rows longer than BFS_HEAVY are expanded by the whole warp.  For each
//                 out-neighbour w: nb = FRONT[v] & ~SEEN[w]; atomicOr into NEXT[w], and the
//                 first writer of a level appends w to the next queue (warp-aggregated);
//   k_bfs_finish  per queued w: new = NEXT[w] & ~SEEN[w]; SEEN |= new; FRONT = new; the
//                 level's OR of all new bits goes to LM[level] (source i is still expanding
//                 at that level), and for a single source DIST[w] = level.
// The eccentricity of source i is the last level whose LM has bit i.  All loop state lives
// on the device, so BFS_BATCH levels are captured once as a CUDA graph and replayed between
// host checks.  The queue counters are double-buffered by the captured level index k: the
// expand of level k reads A[k&1], appends to B[k&1] and zeroes A[(k+1)&1] (read by level
// k-1, appended to by this level's finish); the finish reads B[k&1], appends to A[(k+1)&1]
// and zeroes B[(k+1)&1] -- single writes by one thread, no end-of-kernel atomics.  Kernels
// of a level past the end see an empty queue and return.
#include "common.cuh"
#include "../../include/pasgal_bcc.h"

#include <vector>

namespace pg {

constexpr int BFS_T = 256;
constexpr int BFS_HEAVY = 64;     // rows longer than this are expanded warp-cooperatively
constexpr int BFS_BATCH = 16;     // levels launched per host check

struct BfsWs {
    u64 *SEEN, *FRONT, *NEXT, *LM;
    u32 *QA, *QB;
    u32* cnt;      // [0,1] QA counts A[2], [2,3] QB counts B[2], [4] base level of the replay
    i64 lm_cap;
};

static size_t bfs_carve(BfsWs& b, char* base, i64 n, i64 lm_cap) {
    size_t o = 0;
    auto take = [&](size_t bytes) -> char* {
        o = (o + 255) & ~(size_t)255;
        char* p = base ? base + o : nullptr;
        o += bytes;
        return p;
    };
    const i64 nn = n > 0 ? n : 1;
    b.SEEN = (u64*)take(8 * nn);
    b.FRONT = (u64*)take(8 * nn);
    b.NEXT = (u64*)take(8 * nn);
    b.QA = (u32*)take(4 * nn);
    b.QB = (u32*)take(4 * nn);
    b.cnt = (u32*)take(16);
    b.LM = (u64*)take(8 * lm_cap);
    b.lm_cap = lm_cap;
    return o + 256;
}

// append w to q (counter *cnt) for every lane with `want`, one atomic per warp
__device__ __forceinline__ void bfs_append(bool want, u32 w, u32* q, u32* cnt, int lane) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, want);
    if (!m) return;
    const int lead = __ffs(m) - 1;
    u32 base = 0;
    if (lane == lead) base = atomicAdd(cnt, (u32)__popc(m));
    base = __shfl_sync(0xFFFFFFFFu, base, lead);
    if (want) q[base + __popc(m & ((1u << lane) - 1u))] = w;
}

__device__ __forceinline__ bool bfs_push(u64 f, u32 w, const u64* SEEN, u64* NEXT) {
    const u64 nb = f & ~SEEN[w];
    if (!nb) return false;
    return atomicOr((unsigned long long*)NEXT + w, (unsigned long long)nb) == 0ull;
}

__global__ void __launch_bounds__(BFS_T) k_bfs_expand(const i64* __restrict__ off, const int32_t* __restrict__ tgt,
                                                      const u32* __restrict__ QA, u32* cnt, int k, u64* FRONT,
                                                      const u64* SEEN, u64* NEXT, u32* QB) {
    u32* cnt_next = cnt + 2 + (k & 1);
    const u32 na = cnt[k & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[(k + 1) & 1] = 0;
    const int lane = threadIdx.x & 31;
    const i64 nwarps = (i64)gridDim.x * (BFS_T / 32);
    for (i64 base = ((i64)blockIdx.x * BFS_T + threadIdx.x) & ~31ll; base < na; base += nwarps * 32) {
        const i64 i = base + lane;
        u32 v = 0;
        u64 f = 0;
        i64 a = 0, e = 0;
        if (i < na) {
            v = QA[i];
            f = FRONT[v];
            FRONT[v] = 0;
            a = off[v];
            e = off[(i64)v + 1];
        }
        const bool heavy = e - a > BFS_HEAVY;
        // light rows: lanes in lockstep over their own neighbours
        i64 j = heavy ? e : a;
        for (;;) {
            const bool act = j < e;
            if (!__any_sync(0xFFFFFFFFu, act)) break;
            bool first = false;
            u32 w = 0;
            if (act) {
                w = (u32)tgt[j++];
                first = bfs_push(f, w, SEEN, NEXT);
            }
            bfs_append(first, w, QB, cnt_next, lane);
        }
        // heavy rows: the whole warp strides over each in turn
        unsigned hm = __ballot_sync(0xFFFFFFFFu, heavy);
        while (hm) {
            const int src = __ffs(hm) - 1;
            hm &= hm - 1;
            const u64 fh = __shfl_sync(0xFFFFFFFFu, f, src);
            const i64 ha = __shfl_sync(0xFFFFFFFFu, a, src), he = __shfl_sync(0xFFFFFFFFu, e, src);
            for (i64 k = ha; k < he; k += 32) {
                const i64 s = k + lane;
                bool first = false;
                u32 w = 0;
                if (s < he) {
                    w = (u32)tgt[s];
                    first = bfs_push(fh, w, SEEN, NEXT);
                }
                bfs_append(first, w, QB, cnt_next, lane);
            }
        }
    }
}

// Optional probes: probe[w] = j >= 0 marks vertex w as probe j; the level at which source
// bit i first reaches it is stored in probe_dist[i * nprobe + j] (used by the diameter
// estimate to bound the eccentricities of sources not yet run).
struct BfsProbe {
    const int32_t* probe;
    int32_t* probe_dist;
    i64 nprobe;
};

__global__ void __launch_bounds__(BFS_T) k_bfs_finish(const u32* __restrict__ QB, u32* cnt, int k, u64* SEEN,
                                                      u64* FRONT, u64* NEXT, u32* QA, u64* LM, int32_t* dist,
                                                      BfsProbe pr) {
    u32* cnt_active = cnt + ((k + 1) & 1);
    const u32 nb_ = cnt[2 + (k & 1)];
    const int level = (int)cnt[4] + k + 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[2 + ((k + 1) & 1)] = 0;
    const int lane = threadIdx.x & 31;
    const i64 nwarps = (i64)gridDim.x * (BFS_T / 32);
    u64 lm = 0;
    for (i64 base = ((i64)blockIdx.x * BFS_T + threadIdx.x) & ~31ll; base < nb_; base += nwarps * 32) {
        const i64 i = base + lane;
        bool keep = false;
        u32 w = 0;
        if (i < nb_) {
            w = QB[i];
            const u64 nx = NEXT[w];
            NEXT[w] = 0;
            const u64 s = SEEN[w];
            const u64 nw = nx & ~s;
            if (nw) {
                SEEN[w] = s | nw;
                FRONT[w] = nw;
                lm |= nw;
                keep = true;
                if (dist && (nw & 1ull)) dist[w] = level;
                if (pr.probe) {
                    const int32_t j = pr.probe[w];
                    if (j >= 0) {
                        for (u64 bits = nw; bits; bits &= bits - 1) {
                            const int bit = __ffsll((long long)bits) - 1;
                            pr.probe_dist[(i64)bit * pr.nprobe + j] = level;
                        }
                    }
                }
            }
        }
        bfs_append(keep, w, QA, cnt_active, lane);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) lm |= __shfl_xor_sync(0xFFFFFFFFu, lm, o);
    if (lane == 0 && lm) atomicOr((unsigned long long*)LM + level, (unsigned long long)lm);
}

__global__ void k_bfs_advance(u32* cnt, int by) { cnt[4] += by; }

__global__ void k_bfs_init(i64 n, u64* SEEN, u64* FRONT, u64* NEXT, int32_t* dist) {
    const i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    SEEN[v] = 0;
    FRONT[v] = 0;
    NEXT[v] = 0;
    if (dist) dist[v] = -1;
}

__global__ void k_bfs_sources(const u32* src, int ns, u64* SEEN, u64* FRONT, u32* QA, u32* cnt, int32_t* dist,
                              BfsProbe pr) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    u32 na = 0;
    for (int i = 0; i < ns; ++i) {
        const u32 s = src[i];
        if (SEEN[s] == 0) QA[na++] = s;
        SEEN[s] |= 1ull << i;
        FRONT[s] |= 1ull << i;
        if (dist) dist[s] = 0;
        if (pr.probe && pr.probe[s] >= 0) pr.probe_dist[(i64)i * pr.nprobe + pr.probe[s]] = 0;
    }
    cnt[0] = na;
    cnt[1] = 0;
    cnt[2] = 0;
    cnt[3] = 0;
    cnt[4] = 0;
}

size_t msbfs_workspace_bytes(i64 n, i64 max_levels) {
    BfsWs b;
    return bfs_carve(b, nullptr, n, max_levels + 2);
}

// ecc[i] = eccentricity of sources[i] (max BFS level reached); *levels = levels run.
int msbfs(const pasgal_csr_t* g, const int64_t* sources, int ns, int32_t* dist, int64_t* ecc, int64_t* levels,
          const int32_t* probe, i64 nprobe, int32_t* probe_dist, void* ws, size_t ws_bytes, cudaStream_t st) {
    const BfsProbe pr{nprobe > 0 ? probe : nullptr, probe_dist, nprobe};
    if (pr.probe && !probe_dist) return PASGAL_EINVAL;
    const i64 n = g->n;
    if (ns < 1 || ns > 64 || (dist && ns != 1)) return PASGAL_EINVAL;
    for (int i = 0; i < ns; ++i)
        if (sources[i] < 0 || sources[i] >= n) return PASGAL_ERANGE;
    // LM capacity: every level reaches >= 1 new vertex, so levels < n
    BfsWs b;
    const i64 cap = n + 2;
    if (ws_bytes < bfs_carve(b, nullptr, n, cap)) return PASGAL_EWORKSPACE;
    bfs_carve(b, (char*)ws, n, cap);
    const int B = 256;
    k_bfs_init<<<(unsigned)cdiv(n, B), B, 0, st>>>(n, b.SEEN, b.FRONT, b.NEXT, dist);
    PG_LAUNCH_CHECK();
    u32 hsrc[64];
    for (int i = 0; i < ns; ++i) hsrc[i] = (u32)sources[i];
    u32* dsrc = b.QB;   // the next queue is free until level 1: stage the sources there
    PG_CUDA_TRY(cudaMemcpyAsync(dsrc, hsrc, 4 * ns, cudaMemcpyHostToDevice, st));
    if (pr.probe) PG_CUDA_TRY(cudaMemsetAsync(probe_dist, 0xFF, 4 * (size_t)ns * (size_t)nprobe, st));
    k_bfs_sources<<<1, 32, 0, st>>>(dsrc, ns, b.SEEN, b.FRONT, b.QA, b.cnt, dist, pr);
    PG_LAUNCH_CHECK();
    PG_CUDA_TRY(cudaMemsetAsync(b.LM, 0, 8 * (size_t)cap, st));
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)nsm * 8;
    // BFS_BATCH levels as one graph, captured on a private stream (capture executes
    // nothing, and the caller's stream may be the legacy default stream), launched on st
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cs = nullptr;
    PG_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaError_t ce = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (ce == cudaSuccess) {
        for (int k = 0; k < BFS_BATCH; ++k) {
            k_bfs_expand<<<grid, BFS_T, 0, cs>>>(g->offsets, g->targets, b.QA, b.cnt, k, b.FRONT, b.SEEN, b.NEXT,
                                                 b.QB);
            k_bfs_finish<<<grid, BFS_T, 0, cs>>>(b.QB, b.cnt, k, b.SEEN, b.FRONT, b.NEXT, b.QA, b.LM, dist, pr);
        }
        k_bfs_advance<<<1, 1, 0, cs>>>(b.cnt, BFS_BATCH);
        ce = cudaStreamEndCapture(cs, &graph);
    }
    cudaStreamDestroy(cs);
    if (ce == cudaSuccess) ce = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (ce != cudaSuccess) {
        if (exec) cudaGraphExecDestroy(exec);
        return PASGAL_ECUDA;
    }
    i64 launched = 0;
    u32 h[5] = {0, 0, 0, 0, 0};
    for (;;) {
        ce = cudaGraphLaunch(exec, st);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(h, b.cnt, sizeof h, cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        if (ce != cudaSuccess) break;
        launched += BFS_BATCH;
        if (h[0] == 0 || launched + BFS_BATCH + 2 > cap) break;
    }
    cudaGraphExecDestroy(exec);
    if (ce != cudaSuccess) return PASGAL_ECUDA;
    const i64 level = (i64)h[4] < cap - 1 ? (i64)h[4] : cap - 1;   // levels run (BFS_BATCH is even)
    // eccentricities from the per-level masks
    std::vector<u64> lm((size_t)level + 1);
    PG_CUDA_TRY(cudaMemcpyAsync(lm.data(), b.LM, 8 * (size_t)(level + 1), cudaMemcpyDeviceToHost, st));
    PG_CUDA_TRY(cudaStreamSynchronize(st));
    i64 last = 0;
    for (int i = 0; i < ns; ++i) ecc[i] = 0;
    for (i64 l = 1; l <= level; ++l) {
        if (!lm[l]) continue;
        last = l;
        for (int i = 0; i < ns; ++i)
            if (lm[l] >> i & 1ull) ecc[i] = l;
    }
    if (levels) *levels = last;
    return PASGAL_OK;
}

}  // namespace pg
