// tile.cuh -- merge-path tiles over a CSR: perfectly balanced per-slot work.
//
// The merged sequence of n row-end items and M slot items is cut into tiles of
// TILE_ITEMS items, one CTA per tile, so a tile holds at most TILE_ITEMS slots and at
// most TILE_ITEMS+1 rows whatever the degree skew (RMAT hubs, isolated vertices).  A
// partition pass stores, per tile boundary, the number of rows completed before it.
// Inside a tile every slot learns its row from a shared-memory max-scan of row-start
// marks, so all per-slot loops run slot-strided: a warp touches 32 consecutive slots
// (one 128-byte line of targets) per step.
#pragma once
#include <cub/block/block_scan.cuh>
#include "common.cuh"

namespace pg {

constexpr int TILE_ITEMS = 2048;
constexpr int TILE_BLOCK = 256;
constexpr int TILE_PER_THREAD = TILE_ITEMS / TILE_BLOCK;   // 8
constexpr int TILE_OFF_CLAMP = 4;                          // rows starting > 4 slots before j0 clamp

inline i64 num_tiles(i64 n, i64 m) { return cdiv(n + m, TILE_ITEMS); }

// part[t] = rows completed before merge diagonal t*TILE_ITEMS, t in [0, ntiles]
__global__ void k_tile_partition(const i64* __restrict__ off, i64 n, i64 m, i64 ntiles, u32* __restrict__ part) {
    i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    i64 d = t * TILE_ITEMS;
    if (d > n + m) d = n + m;
    i64 lo = d - m > 0 ? d - m : 0, hi = d < n ? d : n;
    while (lo < hi) {
        i64 mid = (lo + hi + 1) >> 1;
        if (off[mid] <= d - mid) lo = mid; else hi = mid - 1;
    }
    part[t] = (u32)lo;
}

struct TileSmem {
    int off[TILE_ITEMS + 2];      // row start relative to j0, clamped to [-TILE_OFF_CLAMP, TILE_ITEMS+1]
    int srow[TILE_ITEMS];         // local row of each slot
    typename cub::BlockScan<int, TILE_BLOCK>::TempStorage scan;
};

struct Tile {
    i64 j0;       // first slot
    int nslots;   // slots in tile
    i64 i0;       // first row
    int nrows;    // rows touched by the tile's slots or whose end lies in it
};

__device__ __forceinline__ int clamp_rel(i64 x, i64 j0) {
    i64 r = x - j0;
    if (r < -TILE_OFF_CLAMP) r = -TILE_OFF_CLAMP;
    if (r > TILE_ITEMS + 1) r = TILE_ITEMS + 1;
    return (int)r;
}

// Sets up a tile; after return (and the internal __syncthreads), sm.srow[p] is the
// local row of slot j0+p and sm.off[r], sm.off[r+1] bound row i0+r (relative, clamped).
__device__ __forceinline__ Tile tile_setup(const i64* __restrict__ off, i64 n, i64 m,
                                           const u32* __restrict__ part, TileSmem& sm) {
    const int tid = threadIdx.x;
    const i64 t = blockIdx.x;
    Tile tl;
    i64 d0 = t * TILE_ITEMS, d1 = d0 + TILE_ITEMS;
    if (d1 > n + m) d1 = n + m;
    i64 i0 = part[t], i1 = part[t + 1];
    tl.i0 = i0;
    tl.j0 = d0 - i0;
    tl.nslots = (int)((d1 - i1) - tl.j0);
    i64 ilast = i1 < n ? i1 : n - 1;
    tl.nrows = (int)(ilast - i0 + 1);
    if (tl.nrows < 0) tl.nrows = 0;
    for (int r = tid; r <= tl.nrows; r += TILE_BLOCK) sm.off[r] = clamp_rel(off[i0 + r], tl.j0);
    for (int p = tid; p < tl.nslots; p += TILE_BLOCK) sm.srow[p] = 0;
    __syncthreads();
    for (int r = 1 + tid; r < tl.nrows; r += TILE_BLOCK) {
        int s = sm.off[r];
        if (s >= 0 && s < tl.nslots && s < sm.off[r + 1]) sm.srow[s] = r;
    }
    __syncthreads();
    // inclusive max-scan over srow[0, nslots): TILE_PER_THREAD consecutive entries per thread
    int loc[TILE_PER_THREAD];
    int mx = 0;
#pragma unroll
    for (int k = 0; k < TILE_PER_THREAD; ++k) {
        int p = tid * TILE_PER_THREAD + k;
        int v = p < tl.nslots ? sm.srow[p] : 0;
        mx = v > mx ? v : mx;
        loc[k] = mx;
    }
    int excl;
    cub::BlockScan<int, TILE_BLOCK>(sm.scan).ExclusiveScan(mx, excl, 0, cub::Max());
#pragma unroll
    for (int k = 0; k < TILE_PER_THREAD; ++k) {
        int p = tid * TILE_PER_THREAD + k;
        if (p < tl.nslots) sm.srow[p] = loc[k] > excl ? loc[k] : excl;
    }
    __syncthreads();
    return tl;
}

// true iff every slot of local row r lies inside the tile
__device__ __forceinline__ bool tile_row_complete(const TileSmem& sm, const Tile& tl, int r) {
    return sm.off[r] >= 0 && sm.off[r + 1] <= tl.nslots;
}

}  // namespace pg
