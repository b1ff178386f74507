/*
 * pasgal_bcc.h -- C-ABI of the B200-native FAST-BCC library (libpasgal_bcc.so).
 *
 * Drop-in boundary for the reference's biconnectivity entry point
 *   pasgal.oracles.bcc_hopcroft_tarjan(g) -> BccLabels
 *     (/root/reference/pkg/src/pasgal/oracles.py:119-201; output type results.py:45-88)
 * and for the absent parallel `bcc` module it specifies.
 * Plain pointers and sizes only; no torch or CUDA types in the signatures.  Every
 * pointer named "device" is a CUDA device pointer; `stream` is a cudaStream_t passed
 * as void* (NULL = legacy default stream).  All work is stream-ordered and
 * asynchronous unless a function says it synchronises.  The library never allocates
 * device memory: the caller owns inputs, outputs and the workspace.
 *
 * Status codes (mapped by the Python wrapper to the reference's exceptions):
 *   0 PASGAL_OK
 *   1 PASGAL_EINVAL      bad argument           -> ValueError
 *   2 PASGAL_ENOTSYM     not symmetric/simple   -> ValueError("biconnectivity requires a
 *                        symmetric graph")  (oracles.py:127-128)
 *   3 PASGAL_EWORKSPACE  workspace too small    -> ValueError
 *   4 PASGAL_ECUDA       CUDA runtime error     -> RuntimeError
 *   5 PASGAL_EUNSORTED   rows not sorted        -> ValueError
 *   6 PASGAL_ERANGE      target out of range / bad offsets (graph.py:87-96) -> ValueError
 */
#ifndef PASGAL_BCC_H
#define PASGAL_BCC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PASGAL_OK 0
#define PASGAL_EINVAL 1
#define PASGAL_ENOTSYM 2
#define PASGAL_EWORKSPACE 3
#define PASGAL_ECUDA 4
#define PASGAL_EUNSORTED 5
#define PASGAL_ERANGE 6

/* flags for pasgal_bcc */
#define PASGAL_BCC_CANONICAL 1u   /* edge_label = min undirected edge id of the BCC */

/* Symmetric CSR on the device.  Replaces the reference's Graph (graph.py:54-77):
 * offsets int64[n+1] (offsets[n] == m_slots), targets int32[m_slots].
 * Limits: n < 2^31, m_slots < 2^32. */
typedef struct {
    int64_t n;
    int64_t m_slots;
    const int64_t* offsets;   /* device */
    const int32_t* targets;   /* device */
} pasgal_csr_t;

/* Outputs (device).  Replaces BccLabels (results.py:45-66):
 *   edge_label  uint32[m_slots]  one id per BCC, equal on both directions of an edge
 *               (raw: a skeleton component id; CANONICAL: the rank of the BCC's smallest
 *               u<v slot among all u<v slots in CSR order).  Slots of isolated vertices:
 *               none exist.
 *   artic_bits  uint32[ceil(n/32)] articulation bitmap, bit v&31 of word v>>5.
 *   bcc_count   int64 scalar (device).
 *   comp/parent/first  optional uint32[n] (NULL to skip): the parallel-mode fields of
 *               BccLabels (results.py:76-88): skeleton component, spanning-forest parent
 *               (self for roots), preorder rank.
 *   Vertex mode: edge_label may be NULL when comp, parent and first are all given (and
 *   CANONICAL is not set).  The per-slot labelling pass is then skipped and the result is
 *   the O(n) parallel-mode BccLabels ("keeps the result O(n) sized", results.py:49-52):
 *   label(u,w) = comp of the endpoint with the larger first (results.py:80-87). */
typedef struct {
    uint32_t* edge_label;
    uint32_t* artic_bits;
    int64_t* bcc_count;
    uint32_t* comp;
    uint32_t* parent;
    uint32_t* first;
} pasgal_bcc_out_t;

/* Workspace for pasgal_bcc (and pasgal_cc): O(n) words plus one 4-byte row index per
 * 256-slot warp chunk ("O(n) auxiliary space"). */
size_t pasgal_bcc_workspace_bytes(int64_t n, int64_t m_slots);

/* 1 when pasgal_bcc computes the S4 tags of a graph of this size with the two-level kernel
 * (a 4-bit code table kept in L2, exact preorder ranks gathered only for a row's extreme
 * slots) instead of one rank gather per slot: once the rank array (4 bytes per vertex) is
 * at least 4x the device's L2 (2^27 vertices on a B200) and the graph has 8 slots per
 * vertex, or as PASGAL_BCC_TAGS2=0/1 forces.  Reporting only (bench.py names the kernel it timed);
 * results are identical either way. */
int pasgal_bcc_two_level_tags(int64_t n, int64_t m_slots);

/* FAST-BCC on a symmetric, simple CSR with sorted rows.  Asynchronous.  Input is not
 * validated here beyond argument checks; see pasgal_csr_validate.  `seed` perturbs
 * sampling only; canonical outputs are seed-invariant. */
int pasgal_bcc(const pasgal_csr_t* g, const pasgal_bcc_out_t* out, void* workspace,
               size_t workspace_bytes, uint64_t seed, uint32_t flags, void* stream);

/* Stage boundaries for pasgal_bcc_ex profiling: events[k] is recorded on `stream` when
 * stage k ends (events[PASGAL_STAGE_BEGIN] when the call starts).  A single-kernel stage's
 * elapsed time is that kernel's device duration (TAGS = k_tags, LABELS = k_labels). */
#define PASGAL_STAGE_BEGIN 0
#define PASGAL_STAGE_FIRST_CC 1   /* spanning forest: union-find + hook capture        */
#define PASGAL_STAGE_FOREST 2     /* forest CSR + Euler successor                       */
#define PASGAL_STAGE_LISTRANK 3   /* ruling-set list ranking                            */
#define PASGAL_STAGE_TOUR 4       /* tour scatter + preorder scan (first/last/parent)   */
#define PASGAL_STAGE_TAGS 5       /* per-slot min/max of neighbour preorder             */
#define PASGAL_STAGE_RMQ 6        /* low/high, fence test, non-fence tree-edge unions   */
#define PASGAL_STAGE_LAST_CC 7    /* skeleton connectivity over cross edges             */
#define PASGAL_STAGE_ARTIC 8      /* articulation bitmap                                */
#define PASGAL_STAGE_LABELS 9     /* per-slot labels + bcc_count                        */
#define PASGAL_STAGE_CANONICAL 10 /* min-edge-id relabel (only with CANONICAL)          */
#define PASGAL_BCC_NSTAGES 11

typedef struct {
    void** events;   /* cudaEvent_t[n_events] created by the caller (NULL entries skipped) */
    int n_events;
    int launches;    /* out: kernel launches issued by the call */
} pasgal_bcc_prof_t;

/* pasgal_bcc with optional stage events and a launch count (prof may be NULL). */
int pasgal_bcc_ex(const pasgal_csr_t* g, const pasgal_bcc_out_t* out, void* workspace,
                  size_t workspace_bytes, uint64_t seed, uint32_t flags, void* stream,
                  pasgal_bcc_prof_t* prof);

/* CUDA-graph form of pasgal_bcc for repeated calls on fixed buffers (small graphs are
 * launch-bound): _create captures one call's launches for these pointers, sizes, seed and
 * flags (nothing runs); _launch replays it on `stream` -- exactly a pasgal_bcc call on
 * whatever the buffers hold then -- and reports the kernel launches it contains;
 * _destroy frees it.  The buffers must stay allocated while the graph is used. */
typedef struct pasgal_bcc_graph_s* pasgal_bcc_graph_t;
int pasgal_bcc_graph_create(const pasgal_csr_t* g, const pasgal_bcc_out_t* out, void* workspace,
                            size_t workspace_bytes, uint64_t seed, uint32_t flags, pasgal_bcc_graph_t* graph);
int pasgal_bcc_graph_launch(pasgal_bcc_graph_t graph, void* stream, int* launches);
void pasgal_bcc_graph_destroy(pasgal_bcc_graph_t graph);

/* Device validation of the BCC preconditions (graph.py:87-96, 123-158):
 * offsets monotone from 0 to m_slots, targets in [0,n), rows sorted (non-decreasing), and
 * the slot multiset closed under reversal (the k-th copy of w in row u has a k-th copy of
 * u in row w).  Parallel edges are BCC-legal as in the reference (twin pairing); a
 * self-loop slot is left unlabelled (0xFFFFFFFF), as the reference leaves it at -1.
 * SYNCHRONISES `stream`; returns the status (PASGAL_OK, _ERANGE, _EUNSORTED, _ENOTSYM).
 * `workspace` >= pasgal_csr_validate_workspace_bytes(n, m_slots). */
int pasgal_csr_validate(const pasgal_csr_t* g, void* workspace, size_t workspace_bytes,
                        void* stream);

/* pasgal_csr_validate in two halves, so the symmetry check can be scheduled around
 * FAST-BCC.  _begin runs and WAITS FOR the streaming checks (ranges, row order, equal
 * numbers of up and down slots) -- once it returns PASGAL_OK the CSR is safe to pass to
 * pasgal_bcc; a nonzero status is final.  _end launches the bucketed symmetry check on
 * `stream`, waits for it and returns the final status; ordering `stream` after the BCC
 * kernels (an event) lets it run while the labels are copied to the host.  Same workspace
 * for both, untouched in between. */
int pasgal_csr_validate_begin(const pasgal_csr_t* g, void* workspace, size_t workspace_bytes, void* stream);
int pasgal_csr_validate_end(const pasgal_csr_t* g, void* workspace, size_t workspace_bytes, void* stream);
/* The symmetry check of _end without waiting: queued on `stream`, the final status is
 * written to *status (a DEVICE int32) when it completes.  For pipelines that keep several
 * graphs in flight (one workspace per graph in flight). */
int pasgal_csr_validate_check(const pasgal_csr_t* g, void* workspace, size_t workspace_bytes, int32_t* status,
                              void* stream);

/* Workspace for pasgal_csr_validate: 4 bytes per slot (one bucketed 8-byte key per run of
 * "up" slots, at most m/2 of them) plus ~8 KB per CTA of histograms -- O(m), like the
 * reference's twin array (oracles.py:107-116).  This is NOT the size pasgal_bcc needs
 * (pasgal_bcc_workspace_bytes is O(n), ~144 B per vertex): graphs with more than ~36 slots
 * per vertex need more here.  One buffer may serve both calls when they run one after the
 * other on one stream (pasgal_csr_validate has returned before pasgal_bcc is called) if it
 * holds max(pasgal_bcc_workspace_bytes, pasgal_csr_validate_workspace_bytes) bytes. */
size_t pasgal_csr_validate_workspace_bytes(int64_t n, int64_t m_slots);

/* Connected components (SPEC.md:413-420 `connected_components`): the
 * spanning-forest stage of FAST-BCC on its own.  comp[v] = minimum vertex id of v's
 * component (deterministic); *count (device int64) = number of components.  Uses the
 * pasgal_bcc workspace.  Asynchronous. */
int pasgal_cc(const pasgal_csr_t* g, uint32_t* comp, int64_t* count, void* workspace,
              size_t workspace_bytes, uint64_t seed, void* stream);

/* Canonicaliser (results.py:91-112 canonical_edge_partition): relabels
 * any per-slot labelling whose ids lie in [0, label_bound) so that every slot carries the
 * minimum undirected edge id (rank of the u<v slot in CSR order) of its class; ids outside
 * the bound (0xFFFFFFFF = unlabelled) pass through.  Two labellings describe the same
 * partition iff their canonical forms are equal.  labels_out may alias labels_in.  Rows
 * must be sorted.  Asynchronous. */
size_t pasgal_canonicalize_temp_bytes(int64_t n, int64_t m_slots, int64_t label_bound);
int pasgal_canonicalize(const pasgal_csr_t* g, const uint32_t* labels_in, int64_t label_bound,
                        uint32_t* labels_out, void* temp, size_t temp_bytes, void* stream);

/* Positioned error report for a loaded CSR (graph.py:380-395): host_out[0] = first index i
 * with offsets[i-1] > offsets[i] (-1 if none), host_out[1] = first slot whose target lies
 * outside [0, n) (-1 if none).  Used by the .bin loader to raise GraphFormatError with the
 * reference's byte positions.  scratch16: 16 bytes of device memory.  SYNCHRONISES
 * `stream`. */
int pasgal_csr_first_error(const pasgal_csr_t* g, void* scratch16, int64_t* host_out, void* stream);

/* ---------------- device graph construction (north-star subsystem 1) ---------------- */

/* Temp bytes for pasgal_csr_from_keys with `nkeys` keys on n vertices. */
size_t pasgal_csr_build_temp_bytes(int64_t n, int64_t nkeys);

/* Directed edge keys (u<<32 | w) -> sorted, deduplicated CSR with self-loops dropped
 * (the contract of symmetrize/from_edges, graph.py:176-194, 452-481; the keys must
 * already contain both directions).  keys[] and keys_alt[] (both uint64[nkeys]) are
 * clobbered.  offsets int64[n+1]; targets int32 with room for nkeys entries.  Writes the
 * slot count to *m_slots_dev.  Asynchronous. */
int pasgal_csr_from_keys(int64_t n, uint64_t* keys, uint64_t* keys_alt, int64_t nkeys,
                         int64_t* offsets, int32_t* targets, int64_t* m_slots_dev,
                         void* temp, size_t temp_bytes, void* stream);

/* Generators (rules pinned in DESIGN.md "Generators"; host twins in oracle/gen_host.c).
 * draw(seed, c) = sm64(sm64(seed) ^ c), sm64 = the splitmix64 finaliser. */

/* rows x cols 4-neighbour lattice, candidate edge e kept iff draw(seed,e) < keep_threshold
 * (or always when keep_all).  Writes the sorted symmetric CSR directly: offsets int64[n+1],
 * targets int32 (capacity 4*rows*cols), *m_slots_dev.  `temp` >= pasgal_gen_grid_temp_bytes. */
size_t pasgal_gen_grid_temp_bytes(int64_t rows, int64_t cols);
int pasgal_gen_grid(int64_t rows, int64_t cols, uint64_t seed, uint64_t keep_threshold,
                    int keep_all, int64_t* offsets, int32_t* targets, int64_t* m_slots_dev,
                    void* temp, size_t temp_bytes, void* stream);

/* RMAT: `draws` edges on 2^scale vertices; quadrant thresholds ta <= tab <= tabc on 32-bit
 * uniforms.  Emits both directions of every non-loop draw into keys (capacity 2*draws);
 * *nkeys_dev receives the count. */
int pasgal_gen_rmat_keys(int scale, int64_t draws, uint64_t seed, uint32_t ta, uint32_t tab,
                         uint32_t tabc, uint64_t* keys, int64_t* nkeys_dev, void* stream);

/* kNN: npts seeded points with 24-bit coordinates, k nearest (exact integer distance,
 * ties by index, self excluded) on a 2^gbits x 2^gbits cell grid.  Emits both directions
 * of every (i, neighbour) pair into keys (capacity 2*k*npts); *nkeys_dev = 2*k*npts'
 * where npts' accounts for npts <= k.  `temp` >= pasgal_gen_knn_temp_bytes. */
size_t pasgal_gen_knn_temp_bytes(int64_t npts, int gbits);
int pasgal_gen_knn_keys(int64_t npts, int k, uint64_t seed, int gbits, uint64_t* keys,
                        int64_t* nkeys_dev, void* temp, size_t temp_bytes, void* stream);

/* Human-readable status text. */
/* Text adjacency graph files (load_adj, graph.py:250-318) parsed on the
 * device.  The caller puts the raw file bytes in device memory and calls, in order:
 *   pasgal_adj_tokenize        -> number of whitespace-separated tokens (synchronises);
 *   pasgal_adj_token_position  -> {byte, 1-based line} of token k ({nbytes, last line} if
 *                                 k >= ntokens), for header / count tokens and messages;
 *   pasgal_adj_parse           -> offsets int64[n+1] (offsets[n] = m) and targets int32[m]
 *                                 from tokens 3.., given n and m from the header tokens,
 *                                 plus first_err[PASGAL_ADJ_NERR]: per error class the
 *                                 first offending element index (-1: none).  Weights
 *                                 (WeightedAdjacencyGraph) are checked, not stored; a
 *                                 negative weight with a tiny exponent may round to -0.0
 *                                 and is listed in `uncertain` (up to PASGAL_ADJ_UNC_CAP;
 *                                 *n_uncertain is the full count) for the caller to decide.
 * The same temp buffer (pasgal_adj_temp_bytes(nbytes)) must be passed to all three. */
enum {
    PASGAL_ADJ_INV_OFFSET = 0,   /* offset token not an int64 literal */
    PASGAL_ADJ_OVF_OFFSET = 1,   /* offset literal outside int64 */
    PASGAL_ADJ_RANGE_OFFSET = 2, /* offset < 0 or > m */
    PASGAL_ADJ_INV_TARGET = 3,
    PASGAL_ADJ_OVF_TARGET = 4,
    PASGAL_ADJ_RANGE_TARGET = 5, /* target < 0 or >= n */
    PASGAL_ADJ_INV_WEIGHT = 6,   /* weight token not a float literal */
    PASGAL_ADJ_BAD_WEIGHT = 7,   /* weight fails w >= 0 (negative, -inf, nan) */
    PASGAL_ADJ_NERR = 8
};
#define PASGAL_ADJ_UNC_CAP 1024
size_t pasgal_adj_temp_bytes(int64_t nbytes);
int pasgal_adj_tokenize(const uint8_t* text, int64_t nbytes, void* temp, size_t temp_bytes, int64_t* ntokens,
                        void* stream);
int pasgal_adj_token_position(const uint8_t* text, int64_t nbytes, void* temp, size_t temp_bytes, int64_t k,
                              int64_t* byte_line, void* stream);
int pasgal_adj_parse(const uint8_t* text, int64_t nbytes, void* temp, size_t temp_bytes, int64_t n, int64_t m,
                     int weighted, int64_t* offsets, int32_t* targets, int64_t* first_err, int64_t* uncertain,
                     int64_t* n_uncertain, void* stream);

/* Bit-parallel BFS from up to 64 sources at once: the searches of
 * estimate_diameter (graph.py:557-605) and the exact hop distances of bfs_queue
 * (oracles.py:27-46).  Works on any CSR (directed or symmetric); `sources` is a HOST array
 * of nsources in [1, 64] ids in [0, n).  ecc[i] (host) = eccentricity of sources[i] (the
 * largest hop distance it reaches); *levels (host) = the number of BFS levels.  With
 * nsources == 1, `dist` (device int32[n], nullable) receives hop distances, -1 where
 * unreachable.  SYNCHRONISES `stream`.  Workspace: pasgal_msbfs_workspace_bytes(n). */
size_t pasgal_msbfs_workspace_bytes(int64_t n);
int pasgal_msbfs(const pasgal_csr_t* g, const int64_t* sources, int nsources, int32_t* dist, int64_t* ecc,
                 int64_t* levels, void* workspace, size_t workspace_bytes, void* stream);
/* pasgal_msbfs plus probes: probe (device int32[n]) maps a vertex to a probe index in
 * [0, nprobe) or -1; probe_dist (device int32[nsources * nprobe]) receives the hop distance
 * from source i to probe j at [i * nprobe + j], -1 if unreachable. */
int pasgal_msbfs_ex(const pasgal_csr_t* g, const int64_t* sources, int nsources, int32_t* dist, int64_t* ecc,
                    int64_t* levels, const int32_t* probe, int64_t nprobe, int32_t* probe_dist, void* workspace,
                    size_t workspace_bytes, void* stream);

/* VGC frontier engine (SPEC.md vgc-engine run_frontier_loop / local_search, bfs
 * bfs_parallel; PAPER.md "Vertical Granularity Control"), instantiated for
 * exact BFS hop distances from `source` on any CSR (directed or symmetric).  Each round
 * expands the packed frontier by per-warp local searches that process at least `tau`
 * vertices (tau >= 1), possibly many hops deep, with write-min distances; improvements
 * beyond a search's budget form the next frontier.  dist (device int32[n]) = hop distance,
 * -1 if unreachable (oracles.bfs_queue, oracles.py:27-46, exactly); *rounds (host) = rounds
 * executed (tau = 1: the eccentricity of the source + 1).  SYNCHRONISES `stream`.
 * Workspace: pasgal_bfs_vgc_workspace_bytes(n). */
size_t pasgal_bfs_vgc_workspace_bytes(int64_t n);
int pasgal_bfs_vgc(const pasgal_csr_t* g, int64_t source, int tau, int32_t* dist, int64_t* rounds, void* workspace,
                   size_t workspace_bytes, void* stream);
/* pasgal_bfs_vgc with dense rounds (SPEC.md bfs_round_dense): when the graph is symmetric
 * (`symmetric` != 0, the caller's promise) and the frontier's out-degree sum exceeds
 * dense_threshold * m_slots, a round is taken bottom-up (every vertex scans its row for
 * frontier members); identical distances.  *dense_rounds (host, nullable) counts them. */
int pasgal_bfs_vgc_ex(const pasgal_csr_t* g, int64_t source, int tau, double dense_threshold, int symmetric,
                      int32_t* dist, int64_t* rounds, int64_t* dense_rounds, void* workspace, size_t workspace_bytes,
                      void* stream);

/* Articulation bitmap -> one byte per vertex (0/1), on the device: the reference's
 * BccLabels.articulation bool[n] (results.py:45-88) without a host-side bit unpack.
 * Asynchronous on `stream`. */
int pasgal_bits_to_bytes(const uint32_t* bits, int64_t n, uint8_t* bytes, void* stream);

/* Run checksum of a canonical labelling, the device twin of
 * results.canonical_checksum: out[0] = sum over slots s of labels[s] * w(s) mod 2^64 with
 * w(s) = ((s * 0x9E3779B1) mod 2^32) | 1, out[1] = number of set articulation bits.  `out`
 * is DEVICE uint64[2]; bcc_count completes the triple.  Asynchronous. */
int pasgal_canonical_checksum(const uint32_t* labels, int64_t m_slots, const uint32_t* artic_bits, int64_t n,
                              uint64_t* out, void* stream);

const char* pasgal_strerror(int status);

/* Library version string. */
const char* pasgal_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PASGAL_BCC_H */
