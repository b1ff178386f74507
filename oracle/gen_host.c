/*
 * oracle/gen_host.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Host twins of the device graph generators (paper_2404_17101_b200/csrc/gen.cu), used to
 * check that the device generators + device CSR builder emit exactly the CSR the pinned
 * generator rules define, and to build CPU-side test graphs.
 *
 * The reference ships only gen_grid (graph.py:488-508, full lattice, seed ignored) and
 * gen_random (graph.py:511-531); no grid-p, RMAT or kNN generator exists, so the rules
 * are pinned by this repo.  Every CSR here goes through the same
 * symmetrize contract as the reference (graph.py:452-481): both directions, self-loops
 * dropped, duplicates removed, rows sorted.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline uint64_t draw(uint64_t seed, uint64_t ctr) { return sm64(sm64(seed) ^ ctr); }

static int bits_for(int64_t n) { int b = 0; while (b < 63 && ((int64_t)1 << b) < n) ++b; return b ? b : 1; }

/* Directed keys (u<<32|w) -> sorted unique, self-loops dropped -> CSR.  keys[] is clobbered.
 * Returns M (number of slots), or -1 on OOM.  offsets[n+1] int64, targets[M] u32
 * (targets must have room for m_keys entries). */
int64_t host_csr_from_keys(int64_t n, uint64_t* keys, int64_t m_keys,
                           int64_t* offsets, uint32_t* targets) {
    uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(m_keys ? m_keys : 1));
    if (!tmp) return -1;
    int vb = bits_for(n);
    /* keys are (u<<32 | w): sort the w bits [0,vb) and the u bits [32,32+vb) */
    {
        int64_t cnt[256];
        uint64_t* a = keys; uint64_t* b = tmp;
        int shifts[16]; int ns = 0;
        for (int s = 0; s < vb; s += 8) shifts[ns++] = s;
        for (int s = 0; s < vb; s += 8) shifts[ns++] = 32 + s;
        for (int p = 0; p < ns; ++p) {
            int shift = shifts[p];
            memset(cnt, 0, sizeof cnt);
            for (int64_t i = 0; i < m_keys; ++i) cnt[(a[i] >> shift) & 255]++;
            int64_t s = 0;
            for (int d = 0; d < 256; ++d) { int64_t c = cnt[d]; cnt[d] = s; s += c; }
            for (int64_t i = 0; i < m_keys; ++i) b[cnt[(a[i] >> shift) & 255]++] = a[i];
            uint64_t* t = a; a = b; b = t;
        }
        if (a != keys) memcpy(keys, a, sizeof(uint64_t) * (size_t)m_keys);
    }
    free(tmp);
    memset(offsets, 0, sizeof(int64_t) * (size_t)(n + 1));
    int64_t M = 0;
    for (int64_t i = 0; i < m_keys; ++i) {
        if (i && keys[i] == keys[i - 1]) continue;
        uint32_t u = (uint32_t)(keys[i] >> 32), w = (uint32_t)keys[i];
        if (u == w) continue;                      /* symmetrize drops self-loops (graph.py:467-468) */
        offsets[u + 1]++;
        targets[M++] = w;
    }
    for (int64_t v = 0; v < n; ++v) offsets[v + 1] += offsets[v];
    return M;
}

/* ---------------- grid with edge-keep probability ---------------- */
/* Candidate index: horizontal (r,c)-(r,c+1) -> r*(cols-1)+c;
 *                  vertical   (r,c)-(r+1,c) -> rows*(cols-1) + r*cols + c.
 * Kept iff draw(seed, idx) < thr  (thr = floor(p * 2^64); keep_all overrides).
 * Writes the sorted symmetric CSR directly (neighbour order: up, left, right, down). */
static inline int keep(uint64_t seed, uint64_t idx, uint64_t thr, int keep_all) {
    return keep_all || draw(seed, idx) < thr;
}
int64_t host_gen_grid(int64_t rows, int64_t cols, uint64_t seed, uint64_t thr, int keep_all,
                      int64_t* offsets, uint32_t* targets /* capacity 4*rows*cols */) {
    int64_t n = rows * cols, H = rows * (cols - 1), M = 0;
    offsets[0] = 0;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            int64_t v = r * cols + c;
            if (r > 0 && keep(seed, (uint64_t)(H + (r - 1) * cols + c), thr, keep_all)) targets[M++] = (uint32_t)(v - cols);
            if (c > 0 && keep(seed, (uint64_t)(r * (cols - 1) + c - 1), thr, keep_all)) targets[M++] = (uint32_t)(v - 1);
            if (c + 1 < cols && keep(seed, (uint64_t)(r * (cols - 1) + c), thr, keep_all)) targets[M++] = (uint32_t)(v + 1);
            if (r + 1 < rows && keep(seed, (uint64_t)(H + r * cols + c), thr, keep_all)) targets[M++] = (uint32_t)(v + cols);
            offsets[v + 1] = M;
        }
    (void)n;
    return M;
}

/* ---------------- RMAT ---------------- */
/* Draw i, level l (MSB first) uses 32 bits of draw(seed, (i<<5) | (l>>1)): the low half for
 * even l, the high half for odd l.  Quadrant: r < ta -> (0,0); r < tab -> column bit;
 * r < tabc -> row bit; else both.  Edge (row, col); self-loops dropped; both directions. */
int64_t host_rmat_keys(int scale, int64_t draws, uint64_t seed, uint32_t ta, uint32_t tab,
                       uint32_t tabc, uint64_t* keys /* capacity 2*draws */) {
    int64_t k = 0;
    for (int64_t i = 0; i < draws; ++i) {
        uint64_t u = 0, v = 0, w = 0;
        for (int l = 0; l < scale; ++l) {
            if ((l & 1) == 0) w = draw(seed, ((uint64_t)i << 5) | (uint64_t)(l >> 1));
            uint32_t r = (l & 1) ? (uint32_t)(w >> 32) : (uint32_t)w;
            uint64_t bit = 1ull << (scale - 1 - l);
            if (r < ta) { }
            else if (r < tab) v |= bit;
            else if (r < tabc) u |= bit;
            else { u |= bit; v |= bit; }
        }
        if (u == v) continue;
        keys[k++] = (u << 32) | v;
        keys[k++] = (v << 32) | u;
    }
    return k;
}

/* ---------------- kNN on seeded 24-bit points ---------------- */
/* Point i: X = draw(seed, 2i) >> 40, Y = draw(seed, 2i+1) >> 40 (float32 coordinate
 * X * 2^-24 is exact).  Neighbours: the k points j != i minimising (d2, j) with the exact
 * integer d2 = (Xi-Xj)^2 + (Yi-Yj)^2.  Emits both directions of each (i, j). */
void host_knn_points(int64_t npts, uint64_t seed, uint32_t* X, uint32_t* Y) {
    for (int64_t i = 0; i < npts; ++i) {
        X[i] = (uint32_t)(draw(seed, 2 * (uint64_t)i) >> 40);
        Y[i] = (uint32_t)(draw(seed, 2 * (uint64_t)i + 1) >> 40);
    }
}

static inline int better(uint64_t d, uint32_t j, uint64_t bd, uint32_t bj) {
    return d < bd || (d == bd && j < bj);
}

/* cell grid of G x G cells, G = 2^gbits; returns number of keys or -1 */
int64_t host_knn_keys(int64_t npts, int k, const uint32_t* X, const uint32_t* Y, int gbits,
                      uint64_t* keys /* capacity 2*k*npts */) {
    int64_t G = (int64_t)1 << gbits;
    int sh = 24 - gbits;
    int64_t ncell = G * G;
    int64_t* cstart = (int64_t*)calloc((size_t)ncell + 1, sizeof(int64_t));
    uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(npts ? npts : 1));
    if (!cstart || !order) { free(cstart); free(order); return -1; }
    for (int64_t i = 0; i < npts; ++i) cstart[((int64_t)(Y[i] >> sh) * G + (X[i] >> sh)) + 1]++;
    for (int64_t c = 0; c < ncell; ++c) cstart[c + 1] += cstart[c];
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)ncell);
    if (!cur) { free(cstart); free(order); return -1; }
    memcpy(cur, cstart, sizeof(int64_t) * (size_t)ncell);
    for (int64_t i = 0; i < npts; ++i) order[cur[(int64_t)(Y[i] >> sh) * G + (X[i] >> sh)]++] = (uint32_t)i;
    free(cur);
    uint64_t bd[64]; uint32_t bj[64];
    int64_t nk = 0;
    int64_t cs = (int64_t)1 << sh;
    /* points are visited in cell order (neighbouring cells stay cached); the key order
     * does not matter, csr_from_keys sorts them */
    for (int64_t oi = 0; oi < npts; ++oi) {
        int64_t i = order[oi];
        int cnt = 0;
        int64_t cx = X[i] >> sh, cy = Y[i] >> sh;
        for (int64_t r = 0;; ++r) {
            int64_t x0 = cx - r, x1 = cx + r, y0 = cy - r, y1 = cy + r;
            for (int64_t yy = y0; yy <= y1; ++yy) {
                if (yy < 0 || yy >= G) continue;
                for (int64_t xx = x0; xx <= x1; ++xx) {
                    if (xx < 0 || xx >= G) continue;
                    if (r > 0 && yy != y0 && yy != y1 && xx != x0 && xx != x1) continue; /* ring only */
                    int64_t c = yy * G + xx;
                    for (int64_t p = cstart[c]; p < cstart[c + 1]; ++p) {
                        uint32_t j = order[p];
                        if (j == (uint32_t)i) continue;
                        int64_t dx = (int64_t)X[i] - X[j], dy = (int64_t)Y[i] - Y[j];
                        uint64_t d = (uint64_t)(dx * dx + dy * dy);
                        if (cnt < k) {
                            int q = cnt++;
                            while (q > 0 && better(d, j, bd[q - 1], bj[q - 1])) { bd[q] = bd[q - 1]; bj[q] = bj[q - 1]; --q; }
                            bd[q] = d; bj[q] = j;
                        } else if (better(d, j, bd[k - 1], bj[k - 1])) {
                            int q = k - 1;
                            while (q > 0 && better(d, j, bd[q - 1], bj[q - 1])) { bd[q] = bd[q - 1]; bj[q] = bj[q - 1]; --q; }
                            bd[q] = d; bj[q] = j;
                        }
                    }
                }
            }
            /* every point outside the (2r+1)^2 block is at least `lim` away per axis */
            int covers = (x0 <= 0 && y0 <= 0 && x1 >= G - 1 && y1 >= G - 1);
            if (covers) break;
            if (cnt == k) {
                int64_t lim = INT64_MAX;
                if (x0 > 0) { int64_t t = (int64_t)X[i] - x0 * cs; if (t < lim) lim = t; }
                if (x1 < G - 1) { int64_t t = (x1 + 1) * cs - (int64_t)X[i]; if (t < lim) lim = t; }
                if (y0 > 0) { int64_t t = (int64_t)Y[i] - y0 * cs; if (t < lim) lim = t; }
                if (y1 < G - 1) { int64_t t = (y1 + 1) * cs - (int64_t)Y[i]; if (t < lim) lim = t; }
                if (bd[k - 1] < (uint64_t)(lim * lim)) break;
            }
        }
        for (int q = 0; q < cnt; ++q) {
            keys[nk++] = ((uint64_t)i << 32) | bj[q];
            keys[nk++] = ((uint64_t)bj[q] << 32) | (uint64_t)i;
        }
    }
    free(cstart); free(order);
    return nk;
}

/* brute-force kNN (small npts only) used to pin host_knn_keys itself */
int64_t host_knn_keys_brute(int64_t npts, int k, const uint32_t* X, const uint32_t* Y, uint64_t* keys) {
    uint64_t bd[64]; uint32_t bj[64];
    int64_t nk = 0;
    for (int64_t i = 0; i < npts; ++i) {
        int cnt = 0;
        for (int64_t j = 0; j < npts; ++j) {
            if (j == i) continue;
            int64_t dx = (int64_t)X[i] - X[j], dy = (int64_t)Y[i] - Y[j];
            uint64_t d = (uint64_t)(dx * dx + dy * dy);
            if (cnt < k || better(d, (uint32_t)j, bd[k - 1], bj[k - 1])) {
                int q = cnt < k ? cnt++ : k - 1;
                while (q > 0 && better(d, (uint32_t)j, bd[q - 1], bj[q - 1])) { bd[q] = bd[q - 1]; bj[q] = bj[q - 1]; --q; }
                bd[q] = d; bj[q] = (uint32_t)j;
            }
        }
        for (int q = 0; q < cnt; ++q) {
            keys[nk++] = ((uint64_t)i << 32) | bj[q];
            keys[nk++] = ((uint64_t)bj[q] << 32) | (uint64_t)i;
        }
    }
    return nk;
}
