/*
 * oracle/bcc_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the reference's sequential biconnectivity oracle,
 * pasgal.oracles.bcc_hopcroft_tarjan (/root/reference/pkg/src/pasgal/oracles.py:119-201),
 * together with the pieces it calls:
 *   - Graph.is_symmetric -> _same_edge_multiset   (graph.py:123-125, 147-158)
 *   - _twin_edges                                  (oracles.py:107-116)
 * and the parity comparator used on both sides:
 *   - canonical "min undirected edge id per BCC"   (equivalent to results.py:103-112,
 *     see SURVEY.md section 8(b) "Edge-id reading").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_2404_17101_b200) never does.
 *
 * Labels are emitted as int32 (the reference uses int64; comp_count < 2^31 always holds
 * for graphs with fewer than 2^31 undirected edges) to halve host memory at scale.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_NOT_SYMMETRIC 2
#define ORC_NOMEM 5

/* ------------------------------------------------------------------------- */
/* twin + symmetry (oracles.py:107-116, graph.py:147-158)                      */
/* ------------------------------------------------------------------------- */

/* fwd = np.lexsort((dst, src)): slots ordered by (src, dst), stable.  Rows of a
 * CSR are already grouped by src in slot order, so only the within-row order by
 * dst has to be established; it is the identity when the row is sorted. */
static int row_sorted(const uint32_t* t, int64_t a, int64_t b) {
    for (int64_t e = a + 1; e < b; ++e)
        if (t[e - 1] > t[e]) return 0;
    return 1;
}

static const uint32_t* g_sort_tgt;
static int cmp_slot_by_dst(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    uint32_t ta = g_sort_tgt[a], tb = g_sort_tgt[b];
    if (ta != tb) return ta < tb ? -1 : 1;
    return a < b ? -1 : (a > b);            /* stable: tie-break by slot index */
}

/* Computes twin[e] (reverse slot) exactly as the reference's lexsort pairing, and
 * returns 1 iff the edge multiset is closed under reversal (is_symmetric). */
static int twin_and_symmetry(int64_t n, const int64_t* off, const uint32_t* tgt,
                             uint32_t* twin /* [m] */, int* status) {
    int64_t m = off[n];
    *status = ORC_OK;
    if (m == 0) return 1;
    /* fwd = np.lexsort((dst, src)): slots ordered by (src, dst), stable.  Rows of a CSR
     * are already grouped by src, so fwd is the identity unless some row is unsorted;
     * only then is it materialised (int64, per-row stable sort by dst). */
    int sorted_rows = 1;
    for (int64_t u = 0; u < n && sorted_rows; ++u) sorted_rows = row_sorted(tgt, off[u], off[u + 1]);
    int64_t* fwd = NULL;
    if (!sorted_rows) {
        fwd = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
        if (!fwd) { *status = ORC_NOMEM; return 0; }
        for (int64_t e = 0; e < m; ++e) fwd[e] = e;
        for (int64_t u = 0; u < n; ++u) {
            if (!row_sorted(tgt, off[u], off[u + 1])) {
                g_sort_tgt = tgt;
                qsort(fwd + off[u], (size_t)(off[u + 1] - off[u]), sizeof(int64_t), cmp_slot_by_dst);
            }
        }
    }
    /* rev = np.lexsort((src, dst)): order by (dst, src, slot).  A stable counting sort
     * by dst over slots in increasing slot order gives it, because src is
     * non-decreasing in slot order.  Slot ids fit uint32 (m < 2^32). */
    uint32_t* rev = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)m);
    int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    if (!rev || !cnt) { free(fwd); free(rev); free(cnt); *status = ORC_NOMEM; return 0; }
    for (int64_t e = 0; e < m; ++e) {
        if (tgt[e] >= (uint64_t)n) { free(fwd); free(rev); free(cnt); return 0; }
        cnt[tgt[e] + 1]++;
    }
    for (int64_t v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
    for (int64_t e = 0; e < m; ++e) rev[cnt[tgt[e]]++] = (uint32_t)e;
    /* symmetric iff sorted (src,dst) keys == sorted (dst,src) keys, position by position;
     * twin[fwd[k]] = rev[k] (the reference's pairing). */
    /* src of every slot (n < 2^31), so the pairing below reads it with one access */
    uint32_t* src = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)m);
    if (!src) { free(fwd); free(rev); free(cnt); *status = ORC_NOMEM; return 0; }
    for (int64_t v = 0; v < n; ++v)
        for (int64_t e = off[v]; e < off[v + 1]; ++e) src[e] = (uint32_t)v;
    int sym = 1;
    for (int64_t k = 0; k < m && sym; ++k) {
        int64_t ef = fwd ? fwd[k] : k, er = rev[k];
        /* fwd permutes within rows, so src[ef] == src[k] */
        if (src[k] != tgt[er] || tgt[ef] != src[er]) sym = 0;
        twin[ef] = (uint32_t)er;
    }
    free(fwd); free(rev); free(cnt); free(src);
    return sym;
}

int oracle_is_symmetric(int64_t n, const int64_t* off, const uint32_t* tgt) {
    int64_t m = off[n];
    uint32_t* twin = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(m ? m : 1));
    if (!twin) return -ORC_NOMEM;
    int st;
    int sym = twin_and_symmetry(n, off, tgt, twin, &st);
    free(twin);
    if (st) return -st;
    return sym;
}

/* ------------------------------------------------------------------------- */
/* Hopcroft-Tarjan with an explicit edge stack (oracles.py:119-201)            */
/* ------------------------------------------------------------------------- */
/* Returns ORC_OK, ORC_NOT_SYMMETRIC (the reference's ValueError) or ORC_NOMEM.
 * edge_label[m] int32, articulation[n] uint8, *bcc_count. */
int oracle_bcc_hopcroft_tarjan(int64_t n, const int64_t* off, const uint32_t* tgt,
                               int32_t* edge_label, uint8_t* articulation,
                               int64_t* bcc_count) {
    int64_t m = off[n];
    int st = ORC_OK;
    uint32_t* twin = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(m ? m : 1));
    if (!twin) return ORC_NOMEM;
    if (!twin_and_symmetry(n, off, tgt, twin, &st)) {       /* oracles.py:127-128 */
        free(twin);
        return st ? st : ORC_NOT_SYMMETRIC;
    }
    int32_t* disc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));   /* n < 2^31 */
    int32_t* low = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int64_t* frame_v = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t* frame_e = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t* frame_pe = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    uint32_t* estack = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(m ? m : 1));
    if (!disc || !low || !frame_v || !frame_e || !frame_pe || !estack) {
        free(twin); free(disc); free(low); free(frame_v); free(frame_e); free(frame_pe); free(estack);
        return ORC_NOMEM;
    }
    for (int64_t v = 0; v < n; ++v) { disc[v] = -1; low[v] = 0; articulation[v] = 0; }
    for (int64_t e = 0; e < m; ++e) edge_label[e] = -1;
    int32_t timer = 0;
    int64_t comp_count = 0;
    int64_t fs = 0;       /* frame stack size */
    int64_t es = 0;       /* edge stack size */

    for (int64_t root = 0; root < n; ++root) {                /* oracles.py:144 */
        if (disc[root] != -1) continue;
        disc[root] = low[root] = timer++;
        frame_v[fs] = root; frame_e[fs] = off[root]; frame_pe[fs] = -1; ++fs;
        int64_t root_children = 0;
        while (fs) {                                           /* oracles.py:153 */
            int64_t v = frame_v[fs - 1];
            int64_t e = frame_e[fs - 1];
            if (e < off[v + 1]) {
                frame_e[fs - 1] = e + 1;
                int64_t pe = frame_pe[fs - 1];
                if (pe != -1 && e == (int64_t)twin[pe]) continue;   /* oracles.py:159-160 */
                int64_t w = tgt[e];
                if (disc[w] == -1) {                           /* tree edge, oracles.py:162-170 */
                    if (v == root) root_children++;
                    disc[w] = low[w] = timer++;
                    estack[es++] = (uint32_t)e;
                    frame_v[fs] = w; frame_e[fs] = off[w]; frame_pe[fs] = e; ++fs;
                } else if (disc[w] < disc[v]) {                /* back edge, oracles.py:171-174 */
                    estack[es++] = (uint32_t)e;
                    if (disc[w] < low[v]) low[v] = disc[w];
                }
            } else {                                           /* retreat, oracles.py:175-194 */
                --fs;
                int64_t pe = frame_pe[fs];
                if (pe == -1) break;
                int64_t u = frame_v[fs - 1];
                if (low[v] < low[u]) low[u] = low[v];
                if (low[v] >= disc[u]) {
                    if (u != root) articulation[u] = 1;
                    for (;;) {
                        int64_t ee = estack[--es];
                        edge_label[ee] = (int32_t)comp_count;
                        edge_label[twin[ee]] = (int32_t)comp_count;
                        if (ee == pe) break;
                    }
                    comp_count++;
                }
            }
        }
        fs = 0;
        if (root_children >= 2) articulation[root] = 1;        /* oracles.py:195-196 */
    }
    *bcc_count = comp_count;
    free(twin); free(disc); free(low); free(frame_v); free(frame_e); free(frame_pe); free(estack);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* canonical labels: min undirected edge id per BCC                             */
/* ------------------------------------------------------------------------- */
/* The undirected edge id of slot u->w (u<w) is its rank among all u<w slots in CSR
 * order (== key order u*n+w for sorted rows, the order canonical_edge_partition uses,
 * results.py:106-111).  canon_out[s] = min id over the class of label[s].  Labels
 * may be any int32 ids in [0, n_labels); entries < 0 are unlabelled (-> 0xFFFFFFFF).
 * Requires sorted rows.  Returns 0, or ORC_NOMEM. */
int oracle_canonical_min_eid(int64_t n, const int64_t* off, const uint32_t* tgt,
                             const int32_t* label, int64_t n_labels, uint32_t* canon_out) {
    int64_t m = off[n];
    uint32_t* best = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n_labels ? n_labels : 1));
    if (!best) return ORC_NOMEM;
    for (int64_t c = 0; c < n_labels; ++c) best[c] = 0xFFFFFFFFu;
    uint32_t eid = 0;
    for (int64_t u = 0; u < n; ++u)
        for (int64_t s = off[u]; s < off[u + 1]; ++s)
            if ((int64_t)tgt[s] > u) {
                int32_t l = label[s];
                if (l >= 0 && best[l] == 0xFFFFFFFFu) best[l] = eid;   /* first occurrence = min */
                ++eid;
            }
    for (int64_t s = 0; s < m; ++s) canon_out[s] = label[s] >= 0 ? best[label[s]] : 0xFFFFFFFFu;
    free(best);
    return ORC_OK;
}

/* number of undirected (u<w) slots; helper for callers sizing eid arrays */
int64_t oracle_count_upper(int64_t n, const int64_t* off, const uint32_t* tgt) {
    int64_t c = 0;
    for (int64_t u = 0; u < n; ++u)
        for (int64_t s = off[u]; s < off[u + 1]; ++s) c += (int64_t)tgt[s] > u;
    return c;
}

/* ------------------------------------------------------------------------- */
/* connected components (SPEC.md:413-420 `connected_components`; the reference */
/* ships no code for it): BFS from every unvisited vertex in increasing order, */
/* so each component is labelled by its minimum vertex id.                     */
/* ------------------------------------------------------------------------- */
int64_t oracle_connected_components(int64_t n, const int64_t* off, const uint32_t* tgt, int32_t* comp) {
    int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    if (!queue) return -ORC_NOMEM;
    for (int64_t v = 0; v < n; ++v) comp[v] = -1;
    int64_t count = 0;
    for (int64_t r = 0; r < n; ++r) {
        if (comp[r] != -1) continue;
        ++count;
        int64_t head = 0, tail = 0;
        comp[r] = (int32_t)r;
        queue[tail++] = (int32_t)r;
        while (head < tail) {
            int64_t u = queue[head++];
            for (int64_t e = off[u]; e < off[u + 1]; ++e) {
                int64_t w = tgt[e];
                if (comp[w] == -1) {
                    comp[w] = (int32_t)r;
                    queue[tail++] = (int32_t)w;
                }
            }
        }
    }
    free(queue);
    return count;
}

/* ------------------------------------------------------------------------- */
/* FIFO BFS (oracles.bfs_queue, oracles.py:27-46; graph._bfs_ecc, graph.py:557-576):  */
/* dist[v] = hop distance from source, -1 where unreachable; returns the         */
/* eccentricity (largest distance reached), or a negative error.                 */
/* ------------------------------------------------------------------------- */
int64_t oracle_bfs(int64_t n, const int64_t* off, const uint32_t* tgt, int64_t source, int32_t* dist) {
    if (source < 0 || source >= n) return -ORC_NOT_SYMMETRIC - 100;
    int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    if (!queue) return -ORC_NOMEM;
    for (int64_t v = 0; v < n; ++v) dist[v] = -1;
    int64_t head = 0, tail = 0, ecc = 0;
    dist[source] = 0;
    queue[tail++] = (int32_t)source;
    while (head < tail) {
        int64_t u = queue[head++];
        int32_t du = dist[u];
        if (du > ecc) ecc = du;
        for (int64_t e = off[u]; e < off[u + 1]; ++e) {
            int64_t w = tgt[e];
            if (dist[w] == -1) {
                dist[w] = du + 1;
                queue[tail++] = (int32_t)w;
            }
        }
    }
    free(queue);
    return ecc;
}
