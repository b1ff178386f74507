// wchunk.cuh -- warp-chunk iteration over the slots of a CSR (sm_100a).
//
// Every per-slot pass of the pipeline (tags, labels, the union-find passes, canonical
// relabel, validation) runs one warp per chunk of WCH = 32*WCH_U consecutive slots, with
// no shared memory and no block barriers:
//   1. the warp loads its WCH_U target windows (32 consecutive int32 = one 128-byte line
//      each, coalesced) and issues every dependent gather before it needs any result, so
//      each lane keeps WCH_U independent HBM requests in flight;
//   2. slot -> row: the warp holds the ends of the next 32 rows (one coalesced load of
//      offsets) and each lane finds its row with a 6-shuffle binary search; runs of
//      empty rows (isolated RMAT vertices) just repeat the step 32 rows further on;
//   3. rows are contiguous segments of lanes, so per-row reductions are one redux.sync
//      over the segment's lane mask, and only segments cut by a window edge need atomics.
// The chunk's first row comes from a per-chunk partition computed once per call.
#pragma once
#include "common.cuh"

namespace pg {

#ifndef PG_WCH_U
#define PG_WCH_U 8
#endif
constexpr int WCH_U = PG_WCH_U;
constexpr int WCH = 32 * WCH_U;   // slots per warp chunk
constexpr int WCH_BLOCK = 256;    // threads per block (8 warps = 8 chunks)

__host__ __device__ __forceinline__ i64 num_chunks(i64 m) { return cdiv(m, WCH); }
inline unsigned chunk_blocks(i64 m) {
    i64 b = cdiv(num_chunks(m), WCH_BLOCK / 32);
    return (unsigned)(b > 0 ? b : 1);
}

// crow[c] = row containing slot c*WCH (largest r with off[r] <= c*WCH)
__global__ void k_chunk_rows(const i64* __restrict__ off, i64 n, i64 m, i64 nch, u32* __restrict__ crow) {
    i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nch) return;
    i64 s = c * WCH;
    i64 lo = 0, hi = n - 1;
    while (lo < hi) {
        i64 mid = (lo + hi + 1) >> 1;
        if (off[mid] <= s) lo = mid; else hi = mid - 1;
    }
    crow[c] = (u32)lo;
}

// Row of slot s_base+lane for every valid lane (valid lanes are a prefix of the warp).
// `cur` <= row of s_base on entry.  Must be called by all 32 lanes.  Fast path: when the
// current row covers the whole window (long rows: most slots of a power-law graph) one
// broadcast load decides it and no search runs.
__device__ __forceinline__ u32 wc_resolve_row(const i64* __restrict__ off, i64 n, u32 cur, i64 s_base, int lane,
                                              bool valid) {
    if (off[(i64)cur + 1] >= s_base + 32) return cur;   // warp-uniform
    u32 row = 0;
    bool done = !valid;
    u32 c = cur;
    for (;;) {
        i64 e = (i64)c + 1 + lane;
        i64 d = e <= n ? off[e] - s_base : 64;      // end of row c+lane, relative to s_base
        int dr = d < 0 ? 0 : (d > 33 ? 33 : (int)d);
        int pos = 0;                                  // #{l : end(c+l) <= s_base+lane}
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            int v = __shfl_sync(0xFFFFFFFFu, dr, pos + step - 1);
            if (v <= lane) pos += step;
        }
        if (__shfl_sync(0xFFFFFFFFu, dr, pos) <= lane) ++pos;   // the 5 steps reach at most 31
        if (!done && pos < 32) {
            row = c + (u32)pos;
            done = true;
        }
        if (__ballot_sync(0xFFFFFFFFu, !done) == 0u) break;
        c += 32;
    }
    return row;
}

// lane mask of the contiguous segment (equal rows) containing `lane`; sets head/tail info.
struct Seg {
    unsigned mask;
    int lo, hi;         // first / last lane of the segment
    bool cut_left;      // segment starts at lane 0 (row may continue from the previous window)
    bool cut_right;     // segment ends at the window's last valid lane (row may continue)
};

__device__ __forceinline__ Seg wc_segment(u32 row, int lane, bool valid, unsigned validmask) {
    u32 prev = __shfl_up_sync(0xFFFFFFFFu, row, 1);
    bool head = valid && (lane == 0 || prev != row);
    unsigned heads = __ballot_sync(0xFFFFFFFFu, head);
    unsigned le = (lane == 31) ? 0xFFFFFFFFu : ((2u << lane) - 1u);
    Seg s;
    s.lo = 31 - __clz(heads & le);
    unsigned after = heads & ~le;
    int last_valid = 31 - __clz(validmask);
    s.hi = after ? (__ffs(after) - 2) : last_valid;
    s.mask = (s.hi == 31 ? 0xFFFFFFFFu : ((2u << s.hi) - 1u)) & ~((1u << s.lo) - 1u);
    s.cut_left = s.lo == 0;
    s.cut_right = !after;
    return s;
}

}  // namespace pg
