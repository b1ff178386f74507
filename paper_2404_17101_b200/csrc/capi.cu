// capi.cu -- the extern "C" boundary declared in include/pasgal_bcc.h.
#include "common.cuh"
#include "../../include/pasgal_bcc.h"

namespace pg {
int bcc_launch(const pasgal_csr_t* g, const pasgal_bcc_out_t* out, void* ws, size_t ws_bytes, u64 seed, u32 flags,
               cudaStream_t st, pasgal_bcc_prof_t* prof);
size_t bcc_workspace_bytes(i64 n, i64 m);
bool bcc_two_level_tags(i64 n, i64 m);
size_t validate_workspace_bytes(i64 n, i64 m);
int bits_to_bytes(const u32* bits, i64 n, uint8_t* out, cudaStream_t st);
size_t adj_temp_bytes(i64 L);
size_t msbfs_workspace_bytes(i64 n, i64 max_levels);
int msbfs(const pasgal_csr_t* g, const int64_t* sources, int ns, int32_t* dist, int64_t* ecc, int64_t* levels,
          const int32_t* probe, i64 nprobe, int32_t* probe_dist, void* ws, size_t ws_bytes, cudaStream_t st);
int adj_tokenize(const uint8_t* text, i64 L, void* temp, size_t temp_bytes, int64_t* ntokens, cudaStream_t st);
int adj_token_position(const uint8_t* text, i64 L, void* temp, size_t temp_bytes, i64 k, int64_t* byte_line,
                       cudaStream_t st);
int adj_parse(const uint8_t* text, i64 L, void* temp, size_t temp_bytes, i64 n, i64 m, int weighted, i64* offsets,
              int32_t* targets, int64_t* first_err, int64_t* uncertain, int64_t* n_uncertain, cudaStream_t st);
size_t canonicalize_temp_bytes(i64 n, i64 m, i64 nlab);
int canonicalize_launch(const pasgal_csr_t* g, const u32* in, i64 nlab, u32* out, void* temp, size_t temp_bytes,
                        cudaStream_t st);
int csr_first_error(const pasgal_csr_t* g, void* scratch, int64_t* host_out, cudaStream_t st);
int bcc_graph_create(const pasgal_csr_t* g, const pasgal_bcc_out_t* out, void* ws, size_t ws_bytes, u64 seed,
                     uint32_t flags, void** handle);
int bcc_graph_launch(void* handle, cudaStream_t st, int* launches);
void bcc_graph_destroy(void* handle);
size_t vgc_bfs_workspace_bytes(int64_t n);
int vgc_bfs(const pasgal_csr_t* g, int64_t source, int tau, double dense_threshold, int symmetric, int32_t* dist,
            int64_t* rounds, int64_t* dense_rounds, void* ws, size_t ws_bytes, cudaStream_t st);
int canonical_checksum(const uint32_t* lab, int64_t m, const uint32_t* bits, int64_t n, unsigned long long* out,
                       cudaStream_t st);
int cc_launch(const pasgal_csr_t* g, uint32_t* comp, int64_t* count_dev, void* ws, size_t ws_bytes, u64 seed,
              cudaStream_t st);
int csr_validate(const pasgal_csr_t* g, void* ws, size_t ws_bytes, cudaStream_t st);
int csr_validate_begin(const pasgal_csr_t* g, void* ws, size_t ws_bytes, cudaStream_t st);
int csr_validate_end(const pasgal_csr_t* g, void* ws, size_t ws_bytes, cudaStream_t st);
int csr_validate_check(const pasgal_csr_t* g, void* ws, size_t ws_bytes, int32_t* status, cudaStream_t st);
size_t gen_grid_temp_bytes(i64 rows, i64 cols);
int gen_grid(i64 rows, i64 cols, u64 seed, u64 thr, int keep_all, i64* off, int32_t* tgt, i64* m_dev, void* temp,
             size_t temp_bytes, cudaStream_t st);
int gen_rmat_keys(int scale, i64 draws, u64 seed, u32 ta, u32 tab, u32 tabc, u64* keys, i64* nkeys_dev,
                  cudaStream_t st);
size_t gen_knn_temp_bytes(i64 npts, int gbits);
int gen_knn_keys(i64 npts, int k, u64 seed, int gbits, u64* keys, i64* nkeys_dev, void* temp, size_t temp_bytes,
                 cudaStream_t st);
size_t csr_build_temp_bytes(i64 n, i64 nkeys);
int csr_from_keys(i64 n, u64* keys, u64* keys_alt, i64 nkeys, i64* off, int32_t* tgt, i64* m_dev, void* temp,
                  size_t temp_bytes, cudaStream_t st);
}  // namespace pg

static int check_csr(const pasgal_csr_t* g) {
    if (!g) return PASGAL_EINVAL;
    if (g->n < 0 || g->n >= ((int64_t)1 << 31)) return PASGAL_EINVAL;
    if (g->m_slots < 0 || g->m_slots >= ((int64_t)1 << 32)) return PASGAL_EINVAL;
    if (!g->offsets) return PASGAL_EINVAL;
    if (g->m_slots > 0 && !g->targets) return PASGAL_EINVAL;
    return PASGAL_OK;
}

extern "C" {

size_t pasgal_bcc_workspace_bytes(int64_t n, int64_t m_slots) {
    if (n < 0) n = 0;
    if (m_slots < 0) m_slots = 0;
    return pg::bcc_workspace_bytes(n, m_slots);
}

int pasgal_bcc_two_level_tags(int64_t n, int64_t m_slots) { return pg::bcc_two_level_tags(n, m_slots) ? 1 : 0; }

static int check_bcc_args(const pasgal_csr_t* g, const pasgal_bcc_out_t* out, void* workspace, uint32_t flags) {
    int s = check_csr(g);
    if (s) return s;
    if (!out || !out->bcc_count || (g->n > 0 && !out->artic_bits)) return PASGAL_EINVAL;
    // vertex mode (edge_label NULL): the O(n) parallel-mode fields replace the per-slot labels
    const bool vertex_mode = !out->edge_label;
    if (g->m_slots > 0 && vertex_mode &&
        ((flags & PASGAL_BCC_CANONICAL) || (g->n > 0 && (!out->comp || !out->parent || !out->first))))
        return PASGAL_EINVAL;
    if (!workspace) return PASGAL_EWORKSPACE;
    return PASGAL_OK;
}

int pasgal_bcc_ex(const pasgal_csr_t* g, const pasgal_bcc_out_t* out, void* workspace, size_t workspace_bytes,
                  uint64_t seed, uint32_t flags, void* stream, pasgal_bcc_prof_t* prof) {
    int s = check_bcc_args(g, out, workspace, flags);
    if (s) return s;
    return pg::bcc_launch(g, out, workspace, workspace_bytes, seed, flags, (cudaStream_t)stream, prof);
}

int pasgal_bcc_graph_create(const pasgal_csr_t* g, const pasgal_bcc_out_t* out, void* workspace,
                            size_t workspace_bytes, uint64_t seed, uint32_t flags, pasgal_bcc_graph_t* graph) {
    if (!graph) return PASGAL_EINVAL;
    *graph = nullptr;
    int s = check_bcc_args(g, out, workspace, flags);
    if (s) return s;
    void* h = nullptr;
    s = pg::bcc_graph_create(g, out, workspace, workspace_bytes, seed, flags, &h);
    *graph = (pasgal_bcc_graph_t)h;
    return s;
}

int pasgal_bcc_graph_launch(pasgal_bcc_graph_t graph, void* stream, int* launches) {
    if (!graph) return PASGAL_EINVAL;
    return pg::bcc_graph_launch((void*)graph, (cudaStream_t)stream, launches);
}

void pasgal_bcc_graph_destroy(pasgal_bcc_graph_t graph) { pg::bcc_graph_destroy((void*)graph); }

int pasgal_bcc(const pasgal_csr_t* g, const pasgal_bcc_out_t* out, void* workspace, size_t workspace_bytes,
               uint64_t seed, uint32_t flags, void* stream) {
    return pasgal_bcc_ex(g, out, workspace, workspace_bytes, seed, flags, stream, nullptr);
}

int pasgal_cc(const pasgal_csr_t* g, uint32_t* comp, int64_t* count, void* workspace, size_t workspace_bytes,
              uint64_t seed, void* stream) {
    int s = check_csr(g);
    if (s) return s;
    if (!count || (g->n > 0 && !comp)) return PASGAL_EINVAL;
    if (!workspace) return PASGAL_EWORKSPACE;
    return pg::cc_launch(g, comp, count, workspace, workspace_bytes, seed, (cudaStream_t)stream);
}

int pasgal_csr_first_error(const pasgal_csr_t* g, void* scratch16, int64_t* host_out, void* stream) {
    int s = check_csr(g);
    if (s) return s;
    if (!host_out || !scratch16) return PASGAL_EINVAL;
    return pg::csr_first_error(g, scratch16, host_out, (cudaStream_t)stream);
}

size_t pasgal_canonicalize_temp_bytes(int64_t n, int64_t m_slots, int64_t label_bound) {
    return pg::canonicalize_temp_bytes(n < 0 ? 0 : n, m_slots < 0 ? 0 : m_slots, label_bound < 0 ? 0 : label_bound);
}

int pasgal_canonicalize(const pasgal_csr_t* g, const uint32_t* labels_in, int64_t label_bound, uint32_t* labels_out,
                        void* temp, size_t temp_bytes, void* stream) {
    int s = check_csr(g);
    if (s) return s;
    if (label_bound < 0 || label_bound > ((int64_t)1 << 32) || (g->m_slots > 0 && (!labels_in || !labels_out)))
        return PASGAL_EINVAL;
    if (!temp) return PASGAL_EWORKSPACE;
    return pg::canonicalize_launch(g, labels_in, label_bound, labels_out, temp, temp_bytes, (cudaStream_t)stream);
}

int pasgal_csr_validate_begin(const pasgal_csr_t* g, void* workspace, size_t workspace_bytes, void* stream) {
    int s = check_csr(g);
    if (s) return s;
    if (!workspace) return PASGAL_EWORKSPACE;
    return pg::csr_validate_begin(g, workspace, workspace_bytes, (cudaStream_t)stream);
}

int pasgal_csr_validate_end(const pasgal_csr_t* g, void* workspace, size_t workspace_bytes, void* stream) {
    int s = check_csr(g);
    if (s) return s;
    if (!workspace) return PASGAL_EWORKSPACE;
    return pg::csr_validate_end(g, workspace, workspace_bytes, (cudaStream_t)stream);
}

int pasgal_csr_validate_check(const pasgal_csr_t* g, void* workspace, size_t workspace_bytes, int32_t* status,
                              void* stream) {
    int s = check_csr(g);
    if (s) return s;
    if (!workspace) return PASGAL_EWORKSPACE;
    if (!status) return PASGAL_EINVAL;
    return pg::csr_validate_check(g, workspace, workspace_bytes, status, (cudaStream_t)stream);
}

size_t pasgal_csr_validate_workspace_bytes(int64_t n, int64_t m_slots) {
    if (n < 0) n = 0;
    if (m_slots < 0) m_slots = 0;
    return pg::validate_workspace_bytes(n, m_slots);
}

int pasgal_csr_validate(const pasgal_csr_t* g, void* workspace, size_t workspace_bytes, void* stream) {
    int s = check_csr(g);
    if (s) return s;
    if (!workspace) return PASGAL_EWORKSPACE;
    return pg::csr_validate(g, workspace, workspace_bytes, (cudaStream_t)stream);
}

size_t pasgal_csr_build_temp_bytes(int64_t n, int64_t nkeys) { return pg::csr_build_temp_bytes(n, nkeys); }

int pasgal_csr_from_keys(int64_t n, uint64_t* keys, uint64_t* keys_alt, int64_t nkeys, int64_t* offsets,
                         int32_t* targets, int64_t* m_slots_dev, void* temp, size_t temp_bytes, void* stream) {
    if (!offsets || !m_slots_dev || (nkeys > 0 && (!keys || !keys_alt || !targets)) || !temp) return PASGAL_EINVAL;
    return pg::csr_from_keys(n, keys, keys_alt, nkeys, offsets, targets, m_slots_dev, temp, temp_bytes,
                             (cudaStream_t)stream);
}

size_t pasgal_gen_grid_temp_bytes(int64_t rows, int64_t cols) { return pg::gen_grid_temp_bytes(rows, cols); }

int pasgal_gen_grid(int64_t rows, int64_t cols, uint64_t seed, uint64_t keep_threshold, int keep_all,
                    int64_t* offsets, int32_t* targets, int64_t* m_slots_dev, void* temp, size_t temp_bytes,
                    void* stream) {
    if (!offsets || !targets || !m_slots_dev || !temp) return PASGAL_EINVAL;
    return pg::gen_grid(rows, cols, seed, keep_threshold, keep_all, offsets, targets, m_slots_dev, temp, temp_bytes,
                        (cudaStream_t)stream);
}

int pasgal_gen_rmat_keys(int scale, int64_t draws, uint64_t seed, uint32_t ta, uint32_t tab, uint32_t tabc,
                         uint64_t* keys, int64_t* nkeys_dev, void* stream) {
    if ((draws > 0 && !keys) || !nkeys_dev || ta > tab || tab > tabc) return PASGAL_EINVAL;
    return pg::gen_rmat_keys(scale, draws, seed, ta, tab, tabc, keys, nkeys_dev, (cudaStream_t)stream);
}

size_t pasgal_gen_knn_temp_bytes(int64_t npts, int gbits) { return pg::gen_knn_temp_bytes(npts, gbits); }

int pasgal_gen_knn_keys(int64_t npts, int k, uint64_t seed, int gbits, uint64_t* keys, int64_t* nkeys_dev,
                        void* temp, size_t temp_bytes, void* stream) {
    if ((npts > 0 && !keys) || !nkeys_dev || !temp) return PASGAL_EINVAL;
    return pg::gen_knn_keys(npts, k, seed, gbits, keys, nkeys_dev, temp, temp_bytes, (cudaStream_t)stream);
}

size_t pasgal_msbfs_workspace_bytes(int64_t n) {
    if (n < 0) n = 0;
    return pg::msbfs_workspace_bytes(n, n);
}

int pasgal_msbfs(const pasgal_csr_t* g, const int64_t* sources, int nsources, int32_t* dist, int64_t* ecc,
                 int64_t* levels, void* workspace, size_t workspace_bytes, void* stream) {
    int s = check_csr(g);
    if (s) return s;
    if (!sources || !ecc || nsources < 1 || nsources > 64) return PASGAL_EINVAL;
    if (!workspace) return PASGAL_EWORKSPACE;
    return pg::msbfs(g, sources, nsources, dist, ecc, levels, nullptr, 0, nullptr, workspace, workspace_bytes,
                     (cudaStream_t)stream);
}

int pasgal_msbfs_ex(const pasgal_csr_t* g, const int64_t* sources, int nsources, int32_t* dist, int64_t* ecc,
                    int64_t* levels, const int32_t* probe, int64_t nprobe, int32_t* probe_dist, void* workspace,
                    size_t workspace_bytes, void* stream) {
    int s = check_csr(g);
    if (s) return s;
    if (!sources || !ecc || nsources < 1 || nsources > 64 || nprobe < 0) return PASGAL_EINVAL;
    if (!workspace) return PASGAL_EWORKSPACE;
    return pg::msbfs(g, sources, nsources, dist, ecc, levels, probe, nprobe, probe_dist, workspace, workspace_bytes,
                     (cudaStream_t)stream);
}

size_t pasgal_adj_temp_bytes(int64_t nbytes) { return pg::adj_temp_bytes(nbytes < 0 ? 0 : nbytes); }

int pasgal_adj_tokenize(const uint8_t* text, int64_t nbytes, void* temp, size_t temp_bytes, int64_t* ntokens,
                        void* stream) {
    if (nbytes < 0 || (nbytes > 0 && !text) || !ntokens) return PASGAL_EINVAL;
    if (!temp) return PASGAL_EWORKSPACE;
    return pg::adj_tokenize(text, nbytes, temp, temp_bytes, ntokens, (cudaStream_t)stream);
}

int pasgal_adj_token_position(const uint8_t* text, int64_t nbytes, void* temp, size_t temp_bytes, int64_t k,
                              int64_t* byte_line, void* stream) {
    if (nbytes < 0 || (nbytes > 0 && !text) || k < 0 || !byte_line) return PASGAL_EINVAL;
    if (!temp) return PASGAL_EWORKSPACE;
    return pg::adj_token_position(text, nbytes, temp, temp_bytes, k, byte_line, (cudaStream_t)stream);
}

int pasgal_adj_parse(const uint8_t* text, int64_t nbytes, void* temp, size_t temp_bytes, int64_t n, int64_t m,
                     int weighted, int64_t* offsets, int32_t* targets, int64_t* first_err, int64_t* uncertain,
                     int64_t* n_uncertain, void* stream) {
    if (nbytes < 0 || (nbytes > 0 && !text) || n < 0 || n >= ((int64_t)1 << 31) || m < 0 ||
        m >= ((int64_t)1 << 32) || !offsets || (m > 0 && !targets) || !first_err)
        return PASGAL_EINVAL;
    if (!temp) return PASGAL_EWORKSPACE;
    return pg::adj_parse(text, nbytes, temp, temp_bytes, n, m, weighted, offsets, targets, first_err, uncertain,
                         n_uncertain, (cudaStream_t)stream);
}

size_t pasgal_bfs_vgc_workspace_bytes(int64_t n) { return pg::vgc_bfs_workspace_bytes(n < 0 ? 0 : n); }

int pasgal_bfs_vgc_ex(const pasgal_csr_t* g, int64_t source, int tau, double dense_threshold, int symmetric,
                      int32_t* dist, int64_t* rounds, int64_t* dense_rounds, void* workspace, size_t workspace_bytes,
                      void* stream) {
    int s = check_csr(g);
    if (s) return s;
    if (source < 0 || source >= g->n || tau < 1 || !dist || !rounds || !(dense_threshold >= 0.0)) return PASGAL_EINVAL;
    if (!workspace) return PASGAL_EWORKSPACE;
    return pg::vgc_bfs(g, source, tau, dense_threshold, symmetric, dist, rounds, dense_rounds, workspace,
                       workspace_bytes, (cudaStream_t)stream);
}

int pasgal_bfs_vgc(const pasgal_csr_t* g, int64_t source, int tau, int32_t* dist, int64_t* rounds, void* workspace,
                   size_t workspace_bytes, void* stream) {
    return pasgal_bfs_vgc_ex(g, source, tau, 1.0, 0, dist, rounds, nullptr, workspace, workspace_bytes, stream);
}

int pasgal_canonical_checksum(const uint32_t* labels, int64_t m_slots, const uint32_t* artic_bits, int64_t n,
                              uint64_t* out, void* stream) {
    if (n < 0 || m_slots < 0 || !out || (m_slots > 0 && !labels) || (n > 0 && !artic_bits)) return PASGAL_EINVAL;
    return pg::canonical_checksum(labels, m_slots, artic_bits, n, (unsigned long long*)out, (cudaStream_t)stream);
}

int pasgal_bits_to_bytes(const uint32_t* bits, int64_t n, uint8_t* bytes, void* stream) {
    if (n < 0 || (n > 0 && (!bits || !bytes))) return PASGAL_EINVAL;
    return pg::bits_to_bytes(bits, n, bytes, (cudaStream_t)stream);
}

const char* pasgal_strerror(int status) {
    switch (status) {
        case PASGAL_OK: return "ok";
        case PASGAL_EINVAL: return "invalid argument";
        case PASGAL_ENOTSYM: return "biconnectivity requires a symmetric graph";
        case PASGAL_EWORKSPACE: return "workspace too small";
        case PASGAL_ECUDA: return "CUDA error";
        case PASGAL_EUNSORTED: return "adjacency rows must be sorted";
        case PASGAL_ERANGE: return "malformed CSR (offsets or target out of range)";
        default: return "unknown status";
    }
}

const char* pasgal_version(void) { return "pasgal-b200 0.1.0 (sm_100a)"; }

}  // extern "C"
