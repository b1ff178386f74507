// scan.cuh -- single-pass device-wide scan with decoupled look-back (sm_100a).
//
// One CTA per tile of SCAN_BLOCK*SCAN_IPT items; tiles are claimed through an atomic
// counter so every predecessor of a tile is resident or finished (forward progress for
// the look-back spin).  Each tile publishes a 64-bit status word: flag in bits 62-63
// (0 = empty, 1 = tile aggregate, 2 = inclusive prefix) and the value in bits 0-61, so
// flag and value land in one single-copy-atomic store and need no fence.  Values must
// fit in 62 bits.  The look-back is warp-parallel: warp 0 inspects 32 predecessors per
// step and stops at the nearest one holding an inclusive prefix.  Load and store are
// functors, so a scan can be fused with its producer (load) and consumer (store) -- e.g.
// the preorder pass of the rooting stage.  A store must only touch its own tile's items:
// the look-back orders status words, not other tiles' data.
#pragma once
#include <cub/block/block_scan.cuh>
#include "common.cuh"

namespace pg {

constexpr int SCAN_BLOCK = 256;
#ifndef PG_SCAN_IPT
#define PG_SCAN_IPT 8
#endif
constexpr int SCAN_IPT = PG_SCAN_IPT;
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_IPT;
// 32-bit scans: 8 resident tiles per SM (32 registers): without the bound the preorder scan took 56
// registers and ran 4 tiles per SM (C5a tour 10.5 -> 9.8 ms, C3 0.65 -> 0.50).  64-bit scans
// (CSR builder, loaders) keep the compiler's choice: at 32 registers they spill.
#ifndef PG_SCAN_MINB
#define PG_SCAN_MINB 8
#endif
constexpr u64 SCAN_VMASK = (1ull << 62) - 1;

struct SumOp {
    template <class T>
    __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};
struct MinOp {
    template <class T>
    __device__ __forceinline__ T operator()(T a, T b) const { return a < b ? a : b; }
};

// status buffer layout: [0] = tile counter, [1 .. ntiles] = per-tile status
inline size_t scan_status_bytes(i64 nitems) { return sizeof(u64) * (size_t)(cdiv(nitems, SCAN_TILE) + 2); }

template <class T, class Op, class LoadF, class StoreF>
__global__ void __launch_bounds__(SCAN_BLOCK, sizeof(T) == 4 ? PG_SCAN_MINB : 1)
k_scan(i64 nitems, u64* status, T identity, Op op, LoadF load, StoreF store, T* total_out) {
    typedef cub::BlockScan<T, SCAN_BLOCK> BS;
    __shared__ typename BS::TempStorage tmp;
    __shared__ T s_val[SCAN_TILE];
    __shared__ T s_exc[SCAN_TILE];
    __shared__ u32 s_tile;
    __shared__ T s_prefix;
    const int tid = threadIdx.x;
    if (tid == 0) s_tile = (u32)atomicAdd((unsigned long long*)status, 1ull);
    __syncthreads();
    const i64 tile = s_tile;
    const i64 base = tile * SCAN_TILE;
    const i64 ntiles = cdiv(nitems, SCAN_TILE);
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
        i64 idx = base + k * SCAN_BLOCK + tid;
        s_val[k * SCAN_BLOCK + tid] = idx < nitems ? load(idx) : identity;
    }
    __syncthreads();
    T v[SCAN_IPT];
    T acc = identity;
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
        v[k] = s_val[tid * SCAN_IPT + k];
        acc = op(acc, v[k]);
    }
    T excl, total;
    BS(tmp).ExclusiveScan(acc, excl, identity, op, total);
    if (tid < 32) {
        // warp 0 publishes, then looks back over 32 predecessors at a time
        u64* st = status + 1;
        T prefix = identity;
        if (tile == 0) {
            if (tid == 0) st_volatile_u64(st, (2ull << 62) | ((u64)total & SCAN_VMASK));
        } else {
            if (tid == 0) st_volatile_u64(st + tile, (1ull << 62) | ((u64)total & SCAN_VMASK));
            i64 j = tile - 1;   // lane l looks at tile j - l
            for (;;) {
                i64 t = j - tid;
                u64 sv;
                do {
                    sv = t >= 0 ? ld_volatile_u64(st + t) : (2ull << 62);
                } while (__any_sync(0xFFFFFFFFu, (sv >> 62) == 0));
                unsigned inc = __ballot_sync(0xFFFFFFFFu, (sv >> 62) == 2);
                // lanes up to and including the nearest inclusive predecessor contribute
                int last = inc ? __ffs(inc) - 1 : 31;
                T pv = tid <= last ? (T)(sv & SCAN_VMASK) : identity;
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) pv = op(pv, (T)__shfl_xor_sync(0xFFFFFFFFu, pv, o));
                prefix = op(prefix, pv);
                if (inc) break;
                j -= 32;
            }
            if (tid == 0) st_volatile_u64(st + tile, (2ull << 62) | ((u64)op(prefix, total) & SCAN_VMASK));
        }
        if (tid == 0) {
            s_prefix = prefix;
            if (total_out && tile == ntiles - 1) *total_out = op(prefix, total);
        }
    }
    __syncthreads();
    T run = op(s_prefix, excl);
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
        s_exc[tid * SCAN_IPT + k] = run;
        run = op(run, v[k]);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
        i64 idx = base + k * SCAN_BLOCK + tid;
        if (idx < nitems) store(idx, s_exc[k * SCAN_BLOCK + tid], s_val[k * SCAN_BLOCK + tid]);
    }
}

template <class T>
__global__ void k_set_scalar(T* p, T v) { *p = v; }

// Launch a fused scan.  `status` must hold scan_status_bytes(nitems).  For nitems == 0
// the total (if requested) is set to the identity.
template <class T, class Op, class LoadF, class StoreF>
cudaError_t launch_scan(i64 nitems, u64* status, T identity, Op op, LoadF load, StoreF store,
                        T* total_out, cudaStream_t stream, int carveout = -1) {
    if (carveout >= 0) {   // shared-memory carveout preference (percent) of this instantiation
        cudaError_t e = cudaFuncSetAttribute(k_scan<T, Op, LoadF, StoreF>,
                                             cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
        if (e != cudaSuccess) return e;
    }
    if (nitems <= 0) {
        if (total_out) k_set_scalar<T><<<1, 1, 0, stream>>>(total_out, identity);
        return cudaGetLastError();
    }
    i64 ntiles = cdiv(nitems, SCAN_TILE);
    cudaError_t e = cudaMemsetAsync(status, 0, sizeof(u64) * (size_t)(ntiles + 1), stream);
    if (e != cudaSuccess) return e;
    k_scan<T, Op, LoadF, StoreF><<<(unsigned)ntiles, SCAN_BLOCK, 0, stream>>>(nitems, status, identity, op,
                                                                                load, store, total_out);
    return cudaGetLastError();
}

}  // namespace pg
