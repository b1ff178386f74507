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

// targets of chunk c (zeros past the end), streaming loads
__device__ __forceinline__ void wc_load(const int32_t* __restrict__ tgt, i64 m, i64 c, int lane, u32 (&w)[WCH_U]) {
    const i64 s0 = c * WCH;
#pragma unroll
    for (int k = 0; k < WCH_U; ++k) {
        const i64 s = s0 + 32 * k + lane;
        w[k] = s < m ? (u32)__ldcs(tgt + s) : 0u;
    }
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

// --------------------------------------------------------------------------
// Blocked warp chunks: lane l owns the 8 CONSECUTIVE slots s0 + 8l .. s0 + 8l + 7 of the
// warp's 256-slot chunk, so a per-row reduction is a sequential loop in the lane plus one
// segmented warp scan for rows that cross lanes -- instead of a row search, a segment
// mask and two redux per 32-slot window.  Row starts come from one pass over the
// chunk's rows (offsets loaded 32 rows at a time): a per-warp 256-bit start mask and the
// row id at each start position, in shared memory (1 KB + 32 B per warp; no block sync).
// --------------------------------------------------------------------------
namespace pg {

constexpr int BLK_SPL = 8;                 // slots per lane
static_assert(WCH == 32 * BLK_SPL && BLK_SPL == WCH_U, "blocked chunks cover the same 256 slots");

struct BlkSmem {
    union {
        u32 row[WCH];             // row id of a nonempty row starting at chunk position p (where the mask is set)
        u32 xp[WCH + WCH / 32];   // strided -> blocked transpose, padded (conflict-free both ways); dead
                                  // before blk_rows writes `row`
    };
    u32 mask[WCH / 32];
};

// Values gathered in the strided layout (lane l holds positions 32k + l, so the gathers of
// one instruction hit consecutive, often line-sharing, targets) handed to the blocked
// layout (lane l gets positions 8l .. 8l+7).  Padding index p -> p + (p >> 5).
__device__ __forceinline__ void blk_transpose(BlkSmem& sm, int lane, const u32 (&strided)[WCH_U],
                                              u32 (&blocked)[BLK_SPL]) {
    __syncwarp();   // a previous transpose's reads are done before the buffer is rewritten
#pragma unroll
    for (int k = 0; k < WCH_U; ++k) sm.xp[32 * k + lane + k] = strided[k];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < BLK_SPL; ++i) {
        const int p = BLK_SPL * lane + i;
        blocked[i] = sm.xp[p + (p >> 5)];
    }
}

struct BlkRows {
    u32 mb;            // bit i: a nonempty row starts at slot p0 + i of this lane
    u32 r_first;       // row of slot p0
    bool last_open;    // (warp-uniform) the chunk's last row may continue past s1
};

// Row starts of chunk [s0, s1) whose first slot lies in row `base` (the nonempty row
// containing s0): the mask and the row id at each start, in sm.  Returns whether the
// chunk's last row continues past s1.  All 32 lanes call it.
__device__ __forceinline__ bool blk_scan_rows(const i64* __restrict__ off, i64 n, i64 s0, i64 s1, u32 base, int lane,
                                              BlkSmem& sm) {
    __syncwarp();   // the transposes' reads of xp (aliasing row) are done
    if (lane < WCH / 32) sm.mask[lane] = 0u;
    __syncwarp();
    const i64 len = s1 - s0;
    bool last_open = false;
    for (i64 v0 = base;; v0 += 32) {
        const i64 v = v0 + lane;
        const i64 a = v < n ? off[v] : off[n];
        i64 b = __shfl_down_sync(0xFFFFFFFFu, a, 1);
        if (lane == 31) b = v + 1 <= n ? off[v + 1] : off[n];
        const i64 p = a - s0;
        if (b > a && p >= 0 && p < len) {          // a nonempty row starts inside the chunk
            sm.row[p] = (u32)v;
            atomicOr(&sm.mask[p >> 5], 1u << (p & 31));
        }
        // the chunk's last row: the nonempty row containing slot s1 - 1
        const bool holds_last = b > a && a < s1 && b >= s1;
        const unsigned hl = __ballot_sync(0xFFFFFFFFu, holds_last);
        if (hl) last_open = __shfl_sync(0xFFFFFFFFu, b, __ffs(hl) - 1) > s1;
        const i64 bl = __shfl_sync(0xFFFFFFFFu, b, 31);
        if (bl >= s1 || v0 + 32 >= n) break;      // warp-uniform: no later row starts in the chunk
    }
    __syncwarp();
    return last_open;
}

// The blocked view: per lane its start byte and the row of its first slot.
__device__ __forceinline__ BlkRows blk_rows(const i64* __restrict__ off, i64 n, i64 s0, i64 s1, u32 base, int lane,
                                            BlkSmem& sm) {
    const bool last_open = blk_scan_rows(off, n, s0, s1, base, lane, sm);
    BlkRows r;
    const int p0 = BLK_SPL * lane;
    r.mb = (sm.mask[lane >> 2] >> (8 * (lane & 3))) & 0xFFu;
    r.last_open = last_open;
    // row of p0: the last start at or before p0, else base
    u32 rf = base;
    int wi = p0 >> 5;
    u32 bits = sm.mask[wi] & (((p0 & 31) == 31) ? 0xFFFFFFFFu : ((2u << (p0 & 31)) - 1u));
    while (!bits && wi > 0) bits = sm.mask[--wi];
    if (bits) rf = sm.row[32 * wi + 31 - __clz(bits)];
    r.r_first = rf;
    return r;
}

// Segmented inclusive scan over lanes of (mn, mx) with head flags; `started` returns
// whether the segment ending at this lane contains a head (began inside the chunk).
__device__ __forceinline__ void blk_seg_scan(int lane, bool head, u32& mn, u32& mx, bool& started) {
    bool f = head;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 a = __shfl_up_sync(0xFFFFFFFFu, mn, o);
        const u32 b = __shfl_up_sync(0xFFFFFFFFu, mx, o);
        const bool g = __shfl_up_sync(0xFFFFFFFFu, (int)f, o) != 0;
        if (lane >= o && !f) {
            mn = a < mn ? a : mn;
            mx = b > mx ? b : mx;
            f = g;
        }
    }
    started = f;
}

}  // namespace pg
