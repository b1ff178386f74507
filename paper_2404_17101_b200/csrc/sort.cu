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

// temp layout: H u32[256*nsub] | OFF u64[256*nsub] | scan status
size_t radix_sort_temp_bytes(i64 nkeys) {
    i64 cells = (i64)RS_BINS * rs_nsub(nkeys > 0 ? nkeys : 1);
    return ((4 * (size_t)cells + 255) & ~(size_t)255) + ((8 * (size_t)cells + 255) & ~(size_t)255) +
           scan_status_bytes(cells) + 256;
}

// Sorts keys by the bits of `vb`-bit row and column ids; returns the buffer holding the
// result (keys or alt).
cudaError_t radix_sort_edge_keys(u64* keys, u64* alt, i64 nkeys, int vb, void* temp, u64** result,
                                 cudaStream_t st) {
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
