// sort.cu -- LSD radix sort of u64 edge keys for the device CSR builder (sm_100a).
//
// One warp owns a subtile of RS_SUB consecutive keys; no block-level barriers anywhere.
// Per digit pass:
//   1. k_rs_hist    each warp histograms its subtile's digits in a private shared-memory
//                   table (lanes with equal digits aggregated by __match_any_sync), and
//                   writes the 256 counts digit-major: H[d * nsub + sub];
//   2. scan         exclusive prefix over H (decoupled look-back, scan.cuh) -> global
//                   output offset of every (digit, subtile) run; digit-major order makes
//                   the sort stable (runs of one digit follow subtile order);
//   3. k_rs_scatter each warp re-reads its subtile 32 keys at a time, ranks lanes with
//                   equal digits by __match_any_sync (stable within the round) and
//                   scatters to its running per-digit cursors.
// Digits only cover the bits that vary (row bits [32,32+vb), column bits [0,vb)); bits
// vb..31 are zero in every key and the all-ones sentinel sorts last on every digit.
#include <cstdlib>
#include "common.cuh"
#include "scan.cuh"

namespace pg {

constexpr int RS_WARPS = 8;
constexpr int RS_THREADS = RS_WARPS * 32;
constexpr int RS_SUB = 4096;   // keys per warp subtile
constexpr int RS_BINS = 256;
constexpr int RS_U = 4;        // 32-key rounds loaded ahead in the scatter

inline i64 rs_nsub(i64 nkeys) { return cdiv(nkeys, RS_SUB); }

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const u64* __restrict__ keys, i64 nkeys, int shift, u32 mask,
                                                        i64 nsub, u32* __restrict__ H) {
    __shared__ u32 h[RS_WARPS][RS_BINS];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 sub = (i64)blockIdx.x * RS_WARPS + w;
    for (int d = lane; d < RS_BINS; d += 32) h[w][d] = 0;
    __syncwarp();
    if (sub >= nsub) return;
    const i64 a = sub * RS_SUB, b = a + RS_SUB < nkeys ? a + RS_SUB : nkeys;
    for (i64 base = a; base < b; base += 32) {
        i64 i = base + lane;
        bool valid = i < b;
        u32 d = valid ? (u32)(__ldcs(keys + i) >> shift) & mask : 0u;
        unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
        if (valid) {
            unsigned peers = __match_any_sync(vm, d);
            if (lane == __ffs(peers) - 1) h[w][d] += (u32)__popc(peers);   // leaders hold distinct digits
        }
        __syncwarp();
    }
    for (int d = lane; d < RS_BINS; d += 32) H[(i64)d * nsub + sub] = h[w][d];
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const u64* __restrict__ in, u64* __restrict__ out, i64 nkeys,
                                                           int shift, u32 mask, i64 nsub, const u64* __restrict__ OFF) {
    __shared__ u64 cur[RS_WARPS][RS_BINS];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 sub = (i64)blockIdx.x * RS_WARPS + w;
    if (sub >= nsub) return;
    for (int d = lane; d < RS_BINS; d += 32) cur[w][d] = OFF[(i64)d * nsub + sub];
    __syncwarp();
    const i64 a = sub * RS_SUB, b = a + RS_SUB < nkeys ? a + RS_SUB : nkeys;
    const unsigned lt = (1u << lane) - 1u;
    for (i64 base = a; base < b; base += 32 * RS_U) {
        u64 k[RS_U];
#pragma unroll
        for (int j = 0; j < RS_U; ++j) {
            i64 i = base + 32 * j + lane;
            k[j] = i < b ? __ldcs(in + i) : 0ull;
        }
#pragma unroll
        for (int j = 0; j < RS_U; ++j) {
            i64 i = base + 32 * j + lane;
            bool valid = i < b;
            unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
            if (vm == 0u) break;   // warp-uniform
            u32 d = (u32)(k[j] >> shift) & mask;
            unsigned peers = valid ? __match_any_sync(vm, d) : 0u;
            u64 pos = valid ? cur[w][d] + (u64)__popc(peers & lt) : 0ull;
            __syncwarp();
            if (valid && lane == __ffs(peers) - 1) cur[w][d] += (u64)__popc(peers);
            __syncwarp();
            if (valid) out[pos] = k[j];
        }
    }
}

struct HistLoad {
    const u32* H;
    __device__ __forceinline__ u64 operator()(i64 i) const { return H[i]; }
};
struct OffStore {
    u64* OFF;
    __device__ __forceinline__ void operator()(i64 i, u64 ex, u64) const { OFF[i] = ex; }
};

// temp layout (legacy): H u32[256*nsub] | OFF u64[256*nsub] | scan status; onesweep:
// G, GOFF u64[8*256] | tile counters | status u64[ntiles*256]; sized for the larger
static size_t os_temp_bytes(i64 nkeys);
size_t radix_sort_temp_bytes(i64 nkeys) {
    i64 cells = (i64)RS_BINS * rs_nsub(nkeys > 0 ? nkeys : 1);
    const size_t legacy = ((4 * (size_t)cells + 255) & ~(size_t)255) + ((8 * (size_t)cells + 255) & ~(size_t)255) +
                          scan_status_bytes(cells) + 256;
    const size_t os = os_temp_bytes(nkeys) + 256;
    return legacy > os ? legacy : os;
}

// ---------------------------------------------------------------------------------------
// Onesweep form (default): one histogram pass over the keys for every digit, then ONE
// kernel per digit that reads and writes each key once:
//   k_os_hist   global per-digit counts of every pass (shared-memory histograms);
//   k_os_goff   exclusive scan of each pass's 256 counts -> digit bases;
//   k_os_pass   a block takes the next tile of OS_TILE keys (dynamic tile id), ranks them
//               by digit in shared memory (per-warp match_any ranking of 32-key rounds in
//               input order, then an exclusive scan over (digit, warp): stable), publishes
//               its per-digit counts and resolves the counts of all earlier tiles by a
//               decoupled look-back per digit (one thread per digit), stages the tile
//               digit-sorted in shared memory and writes it out: the keys of one digit
//               leave as one contiguous run (~24 keys) instead of per-warp 8-byte scatters
//               that left partially written sectors behind.
// Status words: [63:62] flag (1 aggregate, 2 inclusive prefix), [61:56] pass epoch (a
// word of another pass reads as not yet published), [55:0] count.
// ---------------------------------------------------------------------------------------
#ifndef PG_OS_T
#define PG_OS_T 256
#endif
#ifndef PG_OS_ITEMS
#define PG_OS_ITEMS 16
#endif
#ifndef PG_OS_MINB
#define PG_OS_MINB 3
#endif
constexpr int OS_T = PG_OS_T, OS_W = OS_T / 32, OS_ITEMS = PG_OS_ITEMS, OS_TILE = OS_T * OS_ITEMS, OS_MAXP = 8;
constexpr u64 OS_VMASK = (1ull << 56) - 1;

struct OsPass {
    int shift;
    u32 mask;
};
struct OsPasses {
    OsPass p[OS_MAXP];
    int np;
    int vb;
};

// The bits that vary, packed: row bits [32, 32+vb) above column bits [0, vb), so a
// 2vb-bit key takes ceil(2vb/8) passes (C5a: 7, not 2 x 4).  The all-ones sentinel packs to
// all ones and sorts last.
__device__ __forceinline__ u64 os_vkey(u64 k, int vb) {
    return ((k >> 32) << vb) | (k & ((1ull << vb) - 1));
}

// per-warp shared-memory histograms (plain shared atomics: a power-law graph's hub digits
// collide, and a match_any per key and pass ran at 230 GB/s), merged per block
constexpr int OSH_T = 256, OSH_W = OSH_T / 32;
__global__ void __launch_bounds__(OSH_T) k_os_hist(const u64* __restrict__ keys, i64 nkeys, OsPasses ps,
                                                   unsigned long long* __restrict__ G) {
    extern __shared__ u32 oh[];       // [OSH_W][np][256]
    const int np = ps.np;
    for (int i = threadIdx.x; i < OSH_W * np * RS_BINS; i += OSH_T) oh[i] = 0;
    __syncthreads();
    u32* h = oh + (threadIdx.x >> 5) * np * RS_BINS;
    const i64 stride = (i64)gridDim.x * OSH_T * 4;
    for (i64 base = ((i64)blockIdx.x * OSH_T + threadIdx.x) * 4; base < nkeys; base += stride) {
        u64 k[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) k[j] = base + j < nkeys ? __ldcs(keys + base + j) : 0ull;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (base + j < nkeys) {
#pragma unroll
                for (int q = 0; q < OS_MAXP; ++q)
                    if (q < np)
                        atomicAdd(h + q * RS_BINS + ((u32)(os_vkey(k[j], ps.vb) >> ps.p[q].shift) & ps.p[q].mask), 1u);
            }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < np * RS_BINS; i += OSH_T) {
        u32 c = 0;
        for (int w = 0; w < OSH_W; ++w) c += oh[w * np * RS_BINS + i];
        if (c) atomicAdd(G + i, (unsigned long long)c);
    }
}

__global__ void __launch_bounds__(RS_BINS) k_os_goff(int np, const unsigned long long* __restrict__ G,
                                                     u64* __restrict__ GOFF) {
    __shared__ u64 s[RS_BINS];
    for (int q = 0; q < np; ++q) {
        s[threadIdx.x] = G[q * RS_BINS + threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0) {
            u64 run = 0;
            for (int d = 0; d < RS_BINS; ++d) {
                const u64 c = s[d];
                s[d] = run;
                run += c;
            }
        }
        __syncthreads();
        GOFF[q * RS_BINS + threadIdx.x] = s[threadIdx.x];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(OS_T, PG_OS_MINB) k_os_pass(const u64* __restrict__ in, u64* __restrict__ out, i64 nkeys,
                                                  int vb, int shift, u32 mask, u32 epoch, const u64* __restrict__ GOFF,
                                                  u64* status, u32* tile_ctr) {
    extern __shared__ __align__(16) unsigned char os_smem[];
    u64* sk = (u64*)os_smem;                                  // [OS_TILE] keys, digit-sorted
    u32* wc = (u32*)(sk + OS_TILE);                           // [OS_W][256] per-warp counts -> offsets
    u32* tb = wc + OS_W * RS_BINS;                            // [256] digit base inside the tile (+ scan scratch)
    u64* gb = (u64*)(tb + 3 * RS_BINS + 8);                   // [256] digit base in the output
    __shared__ u32 s_tile;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    for (int d = lane; d < RS_BINS; d += 32) wc[w * RS_BINS + d] = 0;
    __syncthreads();
    const i64 tile = s_tile;
    const i64 t0 = tile * OS_TILE;
    const i64 seg = t0 + (i64)w * 32 * OS_ITEMS;
    u64 k[OS_ITEMS];
    u32 r[OS_ITEMS];
#pragma unroll
    for (int j = 0; j < OS_ITEMS; ++j) {
        const i64 i = seg + 32 * j + lane;
        k[j] = i < nkeys ? __ldcs(in + i) : 0ull;
    }
#pragma unroll
    for (int j = 0; j < OS_ITEMS; ++j) {
        const i64 i = seg + 32 * j + lane;
        const bool valid = i < nkeys;
        const unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
        const u32 d = (u32)(os_vkey(k[j], vb) >> shift) & mask;
        unsigned peers = 0;
        u32 before = 0;
        if (valid) {
            peers = __match_any_sync(vm, d);
            before = wc[w * RS_BINS + d];
        }
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) wc[w * RS_BINS + d] = before + (u32)__popc(peers);
        __syncwarp();
        r[j] = before + (u32)__popc(peers & lt);
    }
    __syncthreads();
    // (digit, warp) exclusive offsets inside the digit, the tile's digit counts and bases
    u32 cnt = 0;
    if (threadIdx.x < RS_BINS) {
        const int d = threadIdx.x;
        for (int q = 0; q < OS_W; ++q) {
            const u32 c = wc[q * RS_BINS + d];
            wc[q * RS_BINS + d] = cnt;
            cnt += c;
        }
        // publish this tile's count early so that later tiles' look-backs can pass it
        const u64 flag = tile == 0 ? 2ull : 1ull;
        st_volatile_u64(status + tile * RS_BINS + d, (flag << 62) | ((u64)epoch << 56) | (u64)cnt);
        // exclusive scan of the 256 tile counts: warp scans + the 8 warp totals
        u32 inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) tb[w] = inc;       // warp totals (tb reused before the final write)
        tb[RS_BINS + 8 + d] = inc - cnt;   // scratch: exclusive inside the warp
    }
    __syncthreads();
    if (threadIdx.x < RS_BINS) {
        const int d = threadIdx.x;
        u32 before = 0;
        for (int q = 0; q < w; ++q) before += tb[q];
        tb[RS_BINS + 8 + RS_BINS + d] = before + tb[RS_BINS + 8 + d];
    }
    __syncthreads();
    if (threadIdx.x < RS_BINS) tb[threadIdx.x] = tb[RS_BINS + 8 + RS_BINS + threadIdx.x];
    if (threadIdx.x < RS_BINS) {  // decoupled look-back per digit
        const int d = threadIdx.x;
        u64 prefix = 0;
        for (i64 t = tile - 1; t >= 0;) {
            const u64 sv = ld_volatile_u64(status + t * RS_BINS + d);
            const u32 f = (u32)(sv >> 62), e = (u32)(sv >> 56) & 63u;
            if (f == 0 || e != epoch) continue;                  // not yet published: spin
            prefix += sv & OS_VMASK;
            if (f == 2) break;
            --t;
        }
        if (tile > 0) st_volatile_u64(status + tile * RS_BINS + d, (2ull << 62) | ((u64)epoch << 56) | (prefix + cnt));
        gb[d] = GOFF[d] + prefix;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < OS_ITEMS; ++j) {
        const i64 i = seg + 32 * j + lane;
        if (i < nkeys) {
            const u32 d = (u32)(os_vkey(k[j], vb) >> shift) & mask;
            sk[tb[d] + wc[w * RS_BINS + d] + r[j]] = k[j];
        }
    }
    __syncthreads();
    const i64 tcount = nkeys - t0 < OS_TILE ? nkeys - t0 : OS_TILE;
    for (int q = threadIdx.x; q < tcount; q += OS_T) {
        const u64 key = sk[q];
        const u32 d = (u32)(os_vkey(key, vb) >> shift) & mask;
        out[gb[d] + (u64)(q - tb[d])] = key;
    }
}

static inline size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }
static inline i64 os_tiles(i64 nkeys) { return cdiv(nkeys > 0 ? nkeys : 1, OS_TILE); }
static size_t os_temp_bytes(i64 nkeys) {
    return al256(8 * (size_t)OS_MAXP * RS_BINS) * 2 + al256(4 * OS_MAXP) + al256(8 * (size_t)os_tiles(nkeys) * RS_BINS);
}
static const size_t OS_SMEM = 8 * (size_t)OS_TILE + 4 * (size_t)OS_W * RS_BINS + 4 * (3 * RS_BINS + 8) + 8 * RS_BINS;

static bool sort_legacy() {
    static const bool legacy = getenv("PASGAL_SORT_LEGACY") != nullptr;
    return legacy;
}

static cudaError_t onesweep_sort(u64* keys, u64* alt, i64 nkeys, int vb, void* temp, u64** result, cudaStream_t st) {
    *result = keys;
    if (nkeys <= 1) return cudaSuccess;
    OsPasses ps{};
    ps.vb = vb;
    for (int bit = 0; bit < 2 * vb; bit += 8) {
        const int width = 2 * vb - bit < 8 ? 2 * vb - bit : 8;
        ps.p[ps.np++] = OsPass{bit, (1u << width) - 1u};
    }
    char* t = (char*)temp;
    unsigned long long* G = (unsigned long long*)t;
    t += al256(8 * (size_t)OS_MAXP * RS_BINS);
    u64* GOFF = (u64*)t;
    t += al256(8 * (size_t)OS_MAXP * RS_BINS);
    u32* ctr = (u32*)t;
    t += al256(4 * OS_MAXP);
    u64* status = (u64*)t;
    const i64 ntiles = os_tiles(nkeys);
    cudaError_t e;
    if ((e = cudaMemsetAsync(G, 0, 8 * (size_t)OS_MAXP * RS_BINS, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(ctr, 0, 4 * OS_MAXP, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(status, 0, 8 * (size_t)ntiles * RS_BINS, st)) != cudaSuccess) return e;
    i64 hb = cdiv(nkeys, 4 * OSH_T);
    if (hb > 148 * 4) hb = 148 * 4;
    const size_t hsm = 4 * (size_t)OSH_W * ps.np * RS_BINS;
    static bool hattr = false;
    if (!hattr) {
        if ((e = cudaFuncSetAttribute(k_os_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(4 * OSH_W * OS_MAXP * RS_BINS))) != cudaSuccess)
            return e;
        hattr = true;
    }
    k_os_hist<<<(unsigned)hb, OSH_T, hsm, st>>>(keys, nkeys, ps, G);
    k_os_goff<<<1, RS_BINS, 0, st>>>(ps.np, G, GOFF);
    static bool attr = false;
    if (!attr) {
        if ((e = cudaFuncSetAttribute(k_os_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)OS_SMEM)) !=
            cudaSuccess)
            return e;
        attr = true;
    }
    u64 *src = keys, *dst = alt;
    for (int q = 0; q < ps.np; ++q) {
        k_os_pass<<<(unsigned)ntiles, OS_T, OS_SMEM, st>>>(src, dst, nkeys, vb, ps.p[q].shift, ps.p[q].mask, (u32)(q + 1),
                                                           GOFF + q * RS_BINS, status, ctr + q);
        u64* tmp = src;
        src = dst;
        dst = tmp;
    }
    *result = src;
    return cudaGetLastError();
}

// Sorts keys by the bits of `vb`-bit row and column ids; returns the buffer holding the
// result (keys or alt).
cudaError_t radix_sort_edge_keys(u64* keys, u64* alt, i64 nkeys, int vb, void* temp, u64** result,
                                 cudaStream_t st) {
    if (!sort_legacy()) return onesweep_sort(keys, alt, nkeys, vb, temp, result, st);
    *result = keys;
    if (nkeys <= 1) return cudaSuccess;
    const i64 nsub = rs_nsub(nkeys);
    const i64 cells = (i64)RS_BINS * nsub;
    char* t = (char*)temp;
    u32* H = (u32*)t;
    t += (4 * (size_t)cells + 255) & ~(size_t)255;
    u64* OFF = (u64*)t;
    t += (8 * (size_t)cells + 255) & ~(size_t)255;
    u64* status = (u64*)t;
    const unsigned grid = (unsigned)cdiv(nsub, RS_WARPS);
    u64 *src = keys, *dst = alt;
    for (int part = 0; part < 2; ++part) {
        const int base = part ? 32 : 0;
        for (int bit = 0; bit < vb; bit += 8) {
            const int width = vb - bit < 8 ? vb - bit : 8;
            const int shift = base + bit;
            const u32 mask = (1u << width) - 1u;
            k_rs_hist<<<grid, RS_THREADS, 0, st>>>(src, nkeys, shift, mask, nsub, H);
            cudaError_t e = launch_scan<u64>(cells, status, 0ull, SumOp(), HistLoad{H}, OffStore{OFF},
                                             (u64*)nullptr, st);
            if (e != cudaSuccess) return e;
            k_rs_scatter<<<grid, RS_THREADS, 0, st>>>(src, dst, nkeys, shift, mask, nsub, OFF);
            u64* tmp = src;
            src = dst;
            dst = tmp;
        }
    }
    *result = src;
    return cudaGetLastError();
}

}  // namespace pg
