// gen.cu -- device graph construction (north-star subsystem 1): seeded generators and the
// CSR builder (own LSD radix sort, sort.cu, + fused dedup/offset scans), replacing the
// reference's host from_edges / symmetrize (graph.py:176-194, 452-481) and gen_grid
// (graph.py:488-508).
// Generator rules are pinned in DESIGN.md "Generators"; host twins: oracle/gen_host.c.
#include "common.cuh"
#include "scan.cuh"
#include "../../include/pasgal_bcc.h"

namespace pg {

size_t radix_sort_temp_bytes(i64 nkeys);
cudaError_t radix_sort_edge_keys(u64* keys, u64* alt, i64 nkeys, int vb, void* temp, u64** result, cudaStream_t st);

constexpr u64 KEY_SENTINEL = ~0ull;   // dropped key (self-loop / missing neighbour)

// ---------------------------------------------------------------------------
// grid with edge-keep probability: CSR written directly, no sort needed
// ---------------------------------------------------------------------------
struct GridSpec {
    i64 rows, cols;
    u64 seed, thr;
    int keep_all;
    __device__ __forceinline__ bool keep(u64 idx) const { return keep_all || draw(seed, idx) < thr; }
    // neighbours of v in sorted order: up, left, right, down
    __device__ __forceinline__ int nbrs(i64 v, u32 out[4]) const {
        i64 r = v / cols, c = v - r * cols, H = rows * (cols - 1);
        int k = 0;
        if (r > 0 && keep((u64)(H + (r - 1) * cols + c))) out[k++] = (u32)(v - cols);
        if (c > 0 && keep((u64)(r * (cols - 1) + c - 1))) out[k++] = (u32)(v - 1);
        if (c + 1 < cols && keep((u64)(r * (cols - 1) + c))) out[k++] = (u32)(v + 1);
        if (r + 1 < rows && keep((u64)(H + r * cols + c))) out[k++] = (u32)(v + cols);
        return k;
    }
};

struct GridDegLoad {
    GridSpec g;
    __device__ __forceinline__ u64 operator()(i64 v) const {
        u32 t[4];
        return (u64)g.nbrs(v, t);
    }
};
struct GridFillStore {
    GridSpec g;
    i64* off;
    int32_t* tgt;
    __device__ __forceinline__ void operator()(i64 v, u64 ex, u64) const {
        u32 t[4];
        int k = g.nbrs(v, t);
        off[v] = (i64)ex;
        for (int q = 0; q < k; ++q) tgt[ex + q] = (int32_t)t[q];
    }
};

__global__ void k_copy_i64(const u64* src, i64* a, i64* b) {
    *a = (i64)*src;
    if (b) *b = (i64)*src;
}

size_t gen_grid_temp_bytes(i64 rows, i64 cols) { return scan_status_bytes(rows * cols) + 256; }

int gen_grid(i64 rows, i64 cols, u64 seed, u64 thr, int keep_all, i64* off, int32_t* tgt, i64* m_dev,
             void* temp, size_t temp_bytes, cudaStream_t st) {
    if (rows < 1 || cols < 1 || rows * cols >= ((i64)1 << 31)) return PASGAL_EINVAL;
    i64 n = rows * cols;
    if (temp_bytes < gen_grid_temp_bytes(rows, cols)) return PASGAL_EWORKSPACE;
    u64* status = (u64*)temp;
    GridSpec g{rows, cols, seed, thr, keep_all};
    // single fused pass: degree -> scan -> write row (offsets + targets)
    PG_CUDA_TRY(launch_scan<u64>(n, status, 0ull, SumOp(), GridDegLoad{g}, GridFillStore{g, off, tgt},
                                 (u64*)(off + n), st));
    k_copy_i64<<<1, 1, 0, st>>>((const u64*)(off + n), m_dev, nullptr);
    PG_LAUNCH_CHECK();
    return PASGAL_OK;
}

// ---------------------------------------------------------------------------
// RMAT
// ---------------------------------------------------------------------------
__global__ void k_rmat(int scale, i64 draws, u64 seed, u32 ta, u32 tab, u32 tabc, u64* keys) {
    i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= draws) return;
    u64 u = 0, v = 0, w = 0;
    for (int l = 0; l < scale; ++l) {
        if ((l & 1) == 0) w = draw(seed, ((u64)i << 5) | (u64)(l >> 1));
        u32 r = (l & 1) ? (u32)(w >> 32) : (u32)w;
        u64 bit = 1ull << (scale - 1 - l);
        if (r < ta) {
        } else if (r < tab) {
            v |= bit;
        } else if (r < tabc) {
            u |= bit;
        } else {
            u |= bit;
            v |= bit;
        }
    }
    ulonglong2 kv;
    if (u == v) {
        kv.x = KEY_SENTINEL;
        kv.y = KEY_SENTINEL;
    } else {
        kv.x = (u << 32) | v;
        kv.y = (v << 32) | u;
    }
    reinterpret_cast<ulonglong2*>(keys)[i] = kv;
}

__global__ void k_set_i64(i64* p, i64 v) { *p = v; }

int gen_rmat_keys(int scale, i64 draws, u64 seed, u32 ta, u32 tab, u32 tabc, u64* keys, i64* nkeys_dev,
                  cudaStream_t st) {
    if (scale < 1 || scale > 31 || draws < 0) return PASGAL_EINVAL;
    if (draws > 0) k_rmat<<<(unsigned)cdiv(draws, 256), 256, 0, st>>>(scale, draws, seed, ta, tab, tabc, keys);
    k_set_i64<<<1, 1, 0, st>>>(nkeys_dev, 2 * draws);
    PG_LAUNCH_CHECK();
    return PASGAL_OK;
}

// ---------------------------------------------------------------------------
// kNN on seeded 24-bit points (exact integer distances, ties by index)
// ---------------------------------------------------------------------------
constexpr int KNN_KMAX = 16;

__global__ void k_knn_points(i64 npts, u64 seed, int gbits, u32* X, u32* Y, u32* CELLCNT, u32* CELL) {
    i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npts) return;
    u32 x = (u32)(draw(seed, 2 * (u64)i) >> 40), y = (u32)(draw(seed, 2 * (u64)i + 1) >> 40);
    X[i] = x;
    Y[i] = y;
    int sh = 24 - gbits;
    u32 c = ((y >> sh) << gbits) | (x >> sh);
    CELL[i] = c;
    atomicAdd(CELLCNT + c, 1u);
}

struct CellLoad {
    const u32* CNT;
    __device__ __forceinline__ u32 operator()(i64 i) const { return CNT[i]; }
};
struct CellStore {
    u32 *START, *CUR;
    __device__ __forceinline__ void operator()(i64 i, u32 ex, u32) const {
        START[i] = ex;
        CUR[i] = ex;
    }
};

__global__ void k_knn_scatter(i64 npts, const u32* CELL, u32* CUR, u32* ORDER) {
    i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npts) return;
    ORDER[atomicAdd(CUR + CELL[i], 1u)] = (u32)i;
}

__device__ __forceinline__ bool knn_better(u64 d, u32 j, u64 bd, u32 bj) { return d < bd || (d == bd && j < bj); }

__global__ void k_knn_query(i64 npts, int k, int gbits, const u32* __restrict__ X, const u32* __restrict__ Y,
                            const u32* __restrict__ START, const u32* __restrict__ ORDER, u64* keys) {
    i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= npts) return;
    const u32 i = ORDER[t];  // process points in cell order for locality
    const i64 G = (i64)1 << gbits;
    const int sh = 24 - gbits;
    const i64 cs = (i64)1 << sh;
    const i64 xi = X[i], yi = Y[i];
    const i64 cx = xi >> sh, cy = yi >> sh;
    const u32 ncell = (u32)(G * G);
    u64 bd[KNN_KMAX];
    u32 bj[KNN_KMAX];
    int cnt = 0;
    for (i64 r = 0;; ++r) {
        i64 x0 = cx - r, x1 = cx + r, y0 = cy - r, y1 = cy + r;
        for (i64 yy = y0; yy <= y1; ++yy) {
            if (yy < 0 || yy >= G) continue;
            bool edge_row = (yy == y0 || yy == y1);
            for (i64 xx = x0; xx <= x1; xx += (edge_row || r == 0) ? 1 : (x1 - x0)) {
                if (xx >= 0 && xx < G) {
                    u32 c = (u32)(yy * G + xx);
                    u32 pe = c + 1 < ncell ? START[c + 1] : (u32)npts;
                    for (u32 p = START[c]; p < pe; ++p) {
                        u32 j = ORDER[p];
                        if (j == i) continue;
                        i64 dx = xi - (i64)X[j], dy = yi - (i64)Y[j];
                        u64 d = (u64)(dx * dx + dy * dy);
                        if (cnt < k || knn_better(d, j, bd[k - 1], bj[k - 1])) {
                            int q = cnt < k ? cnt++ : k - 1;
                            while (q > 0 && knn_better(d, j, bd[q - 1], bj[q - 1])) {
                                bd[q] = bd[q - 1];
                                bj[q] = bj[q - 1];
                                --q;
                            }
                            bd[q] = d;
                            bj[q] = j;
                        }
                    }
                }
                if (x1 == x0) break;
            }
        }
        if (x0 <= 0 && y0 <= 0 && x1 >= G - 1 && y1 >= G - 1) break;
        if (cnt == k) {
            i64 lim = INT64_MAX;
            if (x0 > 0) lim = min(lim, xi - x0 * cs);
            if (x1 < G - 1) lim = min(lim, (x1 + 1) * cs - xi);
            if (y0 > 0) lim = min(lim, yi - y0 * cs);
            if (y1 < G - 1) lim = min(lim, (y1 + 1) * cs - yi);
            if (bd[k - 1] < (u64)(lim * lim)) break;
        }
    }
    u64* o = keys + 2 * (u64)i * k;
    for (int q = 0; q < k; ++q) {
        if (q < cnt) {
            o[2 * q] = ((u64)i << 32) | bj[q];
            o[2 * q + 1] = ((u64)bj[q] << 32) | i;
        } else {
            o[2 * q] = KEY_SENTINEL;
            o[2 * q + 1] = KEY_SENTINEL;
        }
    }
}

struct KnnTemp {
    u32 *X, *Y, *CELL, *CNT, *START, *CUR, *ORDER;
    u64* status;
};
static size_t knn_carve(KnnTemp& t, char* base, i64 npts, int gbits) {
    size_t o = 0;
    auto take = [&](size_t b) -> char* {
        o = (o + 255) & ~(size_t)255;
        char* p = base ? base + o : nullptr;
        o += b;
        return p;
    };
    i64 nc = (i64)1 << (2 * gbits);
    i64 np = npts > 0 ? npts : 1;
    t.X = (u32*)take(4 * np);
    t.Y = (u32*)take(4 * np);
    t.CELL = (u32*)take(4 * np);
    t.ORDER = (u32*)take(4 * np);
    t.CNT = (u32*)take(4 * nc);
    t.START = (u32*)take(4 * nc);
    t.CUR = (u32*)take(4 * nc);
    t.status = (u64*)take(scan_status_bytes(nc));
    return o + 256;
}

size_t gen_knn_temp_bytes(i64 npts, int gbits) {
    KnnTemp t;
    return knn_carve(t, nullptr, npts, gbits);
}

int gen_knn_keys(i64 npts, int k, u64 seed, int gbits, u64* keys, i64* nkeys_dev, void* temp, size_t temp_bytes,
                 cudaStream_t st) {
    if (npts < 0 || npts >= ((i64)1 << 31) || k < 1 || k > KNN_KMAX || gbits < 0 || gbits > 12) return PASGAL_EINVAL;
    if (temp_bytes < gen_knn_temp_bytes(npts, gbits)) return PASGAL_EWORKSPACE;
    KnnTemp t;
    knn_carve(t, (char*)temp, npts, gbits);
    i64 nc = (i64)1 << (2 * gbits);
    k_set_i64<<<1, 1, 0, st>>>(nkeys_dev, 2 * (i64)k * npts);
    if (npts == 0) {
        PG_LAUNCH_CHECK();
        return PASGAL_OK;
    }
    PG_CUDA_TRY(cudaMemsetAsync(t.CNT, 0, 4 * (size_t)nc, st));
    k_knn_points<<<(unsigned)cdiv(npts, 256), 256, 0, st>>>(npts, seed, gbits, t.X, t.Y, t.CNT, t.CELL);
    PG_CUDA_TRY(launch_scan<u32>(nc, t.status, 0u, SumOp(), CellLoad{t.CNT}, CellStore{t.START, t.CUR}, (u32*)nullptr, st));
    k_knn_scatter<<<(unsigned)cdiv(npts, 256), 256, 0, st>>>(npts, t.CELL, t.CUR, t.ORDER);
    k_knn_query<<<(unsigned)cdiv(npts, 128), 128, 0, st>>>(npts, k, gbits, t.X, t.Y, t.START, t.ORDER, keys);
    PG_LAUNCH_CHECK();
    return PASGAL_OK;
}

// ---------------------------------------------------------------------------
// CSR from directed keys: radix sort, unique, drop sentinels/self-loops, row offsets
// ---------------------------------------------------------------------------
static int vbits(i64 n) {
    int b = 1;
    while (b < 32 && ((i64)1 << b) < n) ++b;
    return b;
}

struct UniqLoad {
    const u64* K;
    __device__ __forceinline__ u64 operator()(i64 i) const {
        u64 k = K[i];
        if (k == KEY_SENTINEL || (u32)(k >> 32) == (u32)k) return 0;
        return (i == 0 || K[i - 1] != k) ? 1ull : 0ull;
    }
};
struct UniqStore {
    const u64* K;
    int32_t* tgt;
    i64* off;
    __device__ __forceinline__ void operator()(i64 i, u64 ex, u64 flag) const {
        if (!flag) return;
        u64 k = K[i];
        tgt[ex] = (int32_t)(u32)k;
        u32 u = (u32)(k >> 32);
        // first unique key of its row: the previous key (if any) lies in an earlier row or
        // is a dropped self-loop of this row; find the first kept key of row u
        bool first = true;
        for (i64 j = i - 1; j >= 0; --j) {
            u64 kj = K[j];
            if ((u32)(kj >> 32) != u) break;
            if ((u32)(kj >> 32) != (u32)kj) { first = false; break; }
        }
        if (first) off[u] = (i64)ex;
    }
};

__global__ void k_fill_i64(i64* p, i64 count, i64 v) {
    i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) p[i] = v;
}

// offsets[v] = min(offsets[v..n]) by a reversed min-scan (empty rows inherit the next start)
struct RevLoad {
    const i64* off;
    i64 n;
    __device__ __forceinline__ u64 operator()(i64 i) const { return (u64)off[n - i]; }
};
struct RevStore {
    i64* off;
    i64 n;
    __device__ __forceinline__ void operator()(i64 i, u64 ex, u64 v) const { off[n - i] = (i64)(ex < v ? ex : v); }
};

size_t csr_build_temp_bytes(i64 n, i64 nkeys) {
    size_t srt = radix_sort_temp_bytes(nkeys > 0 ? nkeys : 1);
    size_t sc = scan_status_bytes(nkeys > n + 1 ? nkeys : n + 1);
    return ((srt + 255) & ~(size_t)255) + sc + 512;
}

int csr_from_keys(i64 n, u64* keys, u64* keys_alt, i64 nkeys, i64* off, int32_t* tgt, i64* m_dev, void* temp,
                  size_t temp_bytes, cudaStream_t st) {
    if (n < 0 || n >= ((i64)1 << 31) || nkeys < 0) return PASGAL_EINVAL;
    if (temp_bytes < csr_build_temp_bytes(n, nkeys)) return PASGAL_EWORKSPACE;
    size_t srt = radix_sort_temp_bytes(nkeys > 0 ? nkeys : 1);
    u64* status = (u64*)((char*)temp + ((srt + 255) & ~(size_t)255));
    u64* sorted = keys;
    if (nkeys > 0) PG_CUDA_TRY(radix_sort_edge_keys(keys, keys_alt, nkeys, vbits(n), temp, &sorted, st));
    // offsets[0..n-1] = "none yet"; offsets[n] = M (set by the unique scan's total)
    k_fill_i64<<<(unsigned)cdiv(n + 1, 256), 256, 0, st>>>(off, n + 1, (i64)SCAN_VMASK);
    PG_CUDA_TRY(launch_scan<u64>(nkeys, status, 0ull, SumOp(), UniqLoad{sorted}, UniqStore{sorted, tgt, off},
                                 (u64*)(off + n), st));
    PG_CUDA_TRY(launch_scan<u64>(n + 1, status, (u64)SCAN_VMASK, MinOp(), RevLoad{off, n}, RevStore{off, n},
                                 (u64*)nullptr, st));
    k_copy_i64<<<1, 1, 0, st>>>((const u64*)(off + n), m_dev, nullptr);
    PG_LAUNCH_CHECK();
    return PASGAL_OK;
}

}  // namespace pg
