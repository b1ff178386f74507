// adj.cu -- device tokenizer / parser for the reference's text adjacency format
// (pasgal.graph.load_adj, graph.py:250-318): "AdjacencyGraph | WeightedAdjacencyGraph",
// n, m, n offsets, m targets [, m weights], separated by ASCII whitespace (bytes.split()).
//
// The file goes to HBM as raw bytes and is processed in 4 KB tiles (256 threads x 16 bytes,
// one 16-byte load per thread):
//   k_adj_count   token starts per tile (a start = non-space byte after a space or at 0);
//   launch_scan   exclusive scan of the tile counts -> token index of each tile's first start;
//   k_adj_parse   re-counts per thread, block-scans to the token index of every start, and
//                 the thread owning a start parses that token straight into the int64
//                 offsets / int32 targets (weights are only checked: BCC is unweighted).
// Errors are not raised here: for each error class the first offending element index is
// kept with atomicMin, and the host applies them in the reference's order with its
// messages (the token's line and byte come from k_adj_find + k_adj_count_nl).
// Numeric grammar = numpy's conversion of bytes tokens (Python int()/float()):
//   int   [+-]? D (_? D)*                 (int64 range, else OverflowError)
//   float [+-]? (inf|infinity|nan)  |  [+-]? (P(.P?)? | .P) ([eE][+-]?P)?,  P = D(_?D)*
#include "common.cuh"
#include "scan.cuh"
#include "../../include/pasgal_bcc.h"

namespace pg {

constexpr int ADJ_THREADS = 256, ADJ_BPT = 16, ADJ_TILE = ADJ_THREADS * ADJ_BPT;

__device__ __forceinline__ bool adj_ws(u32 c) { return c == 0x20u || (c >= 0x09u && c <= 0x0Du); }
__device__ __forceinline__ bool adj_digit(u32 c) { return c - '0' < 10u; }

// the 16 bytes of thread slot b0 (b0 % 16 == 0) as four words; bytes past L read as spaces
__device__ __forceinline__ uint4 adj_load16(const uint8_t* d, i64 L, i64 b0) {
    if (b0 + 16 <= L) return *reinterpret_cast<const uint4*>(d + b0);
    u32 w[4] = {0x20202020u, 0x20202020u, 0x20202020u, 0x20202020u};
    for (int k = 0; k < 16 && b0 + k < L; ++k) {
        w[k >> 2] = (w[k >> 2] & ~(0xFFu << (8 * (k & 3)))) | ((u32)d[b0 + k] << (8 * (k & 3)));
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// bit k set iff byte b0+k starts a token
__device__ __forceinline__ u32 adj_starts(const uint8_t* d, i64 L, i64 b0) {
    const uint4 v = adj_load16(d, L, b0);
    const u32 w[4] = {v.x, v.y, v.z, v.w};
    bool prev_ws = b0 == 0 ? true : (b0 - 1 < L ? adj_ws(d[b0 - 1]) : true);
    u32 mask = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const bool s = adj_ws((w[k >> 2] >> (8 * (k & 3))) & 0xFFu);
        if (!s && prev_ws && b0 + k < L) mask |= 1u << k;
        prev_ws = s;
    }
    return mask;
}

__global__ void __launch_bounds__(ADJ_THREADS) k_adj_count(const uint8_t* __restrict__ d, i64 L, u64* tcnt) {
    __shared__ u32 s_w[ADJ_THREADS / 32];
    const i64 b0 = (i64)blockIdx.x * ADJ_TILE + (i64)threadIdx.x * ADJ_BPT;
    u32 c = b0 < L ? (u32)__popc(adj_starts(d, L, b0)) : 0u;
    c = __reduce_add_sync(0xFFFFFFFFu, c);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        u32 t = 0;
        for (int i = 0; i < ADJ_THREADS / 32; ++i) t += s_w[i];
        tcnt[blockIdx.x] = t;
    }
}

struct AdjLoad {
    const u64* c;
    __device__ __forceinline__ u64 operator()(i64 i) const { return c[i]; }
};
struct AdjStore {
    u64* o;
    __device__ __forceinline__ void operator()(i64 i, u64 ex, u64) const { o[i] = ex; }
};

// token [p, end): end = first whitespace at or after p (or L)
__device__ __forceinline__ i64 adj_tok_end(const uint8_t* d, i64 L, i64 p) {
    while (p < L && !adj_ws(d[p])) ++p;
    return p;
}

// 0 = invalid syntax, 1 = ok, 2 = syntax ok but outside int64 (OverflowError)
__device__ int adj_parse_int(const uint8_t* d, i64 p, i64 end, i64* out) {
    bool neg = false;
    if (p < end && (d[p] == '+' || d[p] == '-')) {
        neg = d[p] == '-';
        ++p;
    }
    if (p >= end || !adj_digit(d[p])) return 0;
    const u64 lim = neg ? (1ull << 63) : (1ull << 63) - 1;
    u64 acc = 0;
    bool ovf = false;
    for (; p < end; ++p) {
        const u32 c = d[p];
        if (c == '_') {
            if (p + 1 >= end || !adj_digit(d[p + 1])) return 0;   // '_' only between digits
            continue;
        }
        if (!adj_digit(c)) return 0;
        const u64 dig = c - '0';
        if (!ovf && acc > (lim - dig) / 10) ovf = true;
        if (!ovf) acc = acc * 10 + dig;
    }
    if (ovf) return 2;
    *out = neg ? (i64)(0ull - acc) : (i64)acc;
    return 1;
}

// digit part D(_?D)* starting at p: returns the end, counts digits, notes the first nonzero
__device__ __forceinline__ i64 adj_digits(const uint8_t* d, i64 p, i64 end, int* ndig, int* first_nz) {
    *ndig = 0;
    *first_nz = -1;
    while (p < end) {
        const u32 c = d[p];
        if (adj_digit(c)) {
            if (c != '0' && *first_nz < 0) *first_nz = *ndig;
            ++*ndig;
            ++p;
        } else if (c == '_' && *ndig > 0 && p + 1 < end && adj_digit(d[p + 1])) {
            ++p;
        } else {
            break;
        }
    }
    return p;
}

__device__ __forceinline__ bool adj_word(const uint8_t* d, i64 p, i64 end, const char* w) {
    i64 k = 0;
    for (; w[k]; ++k)
        if (p + k >= end || (d[p + k] | 0x20u) != (u32)w[k]) return false;
    return p + k == end;
}

// weight token class: 0 invalid, 1 ok (>= 0, incl. -0.0 and +inf), 2 fails ~(w >= 0)
// (negative non-zero, -inf, nan), 3 negative with a tiny exponent: the host decides
// whether it rounds to -0.0
__device__ int adj_weight_class(const uint8_t* d, i64 p, i64 end) {
    bool neg = false;
    if (p < end && (d[p] == '+' || d[p] == '-')) {
        neg = d[p] == '-';
        ++p;
    }
    if (adj_word(d, p, end, "inf") || adj_word(d, p, end, "infinity")) return neg ? 2 : 1;
    if (adj_word(d, p, end, "nan")) return 2;
    int ni, nzi, nf = 0, nzf = -1;
    p = adj_digits(d, p, end, &ni, &nzi);
    if (p < end && d[p] == '.') {
        ++p;
        p = adj_digits(d, p, end, &nf, &nzf);
    }
    if (ni + nf == 0) return 0;
    long long ex = 0;
    if (p < end && (d[p] == 'e' || d[p] == 'E')) {
        ++p;
        bool eneg = false;
        if (p < end && (d[p] == '+' || d[p] == '-')) {
            eneg = d[p] == '-';
            ++p;
        }
        if (p >= end || !adj_digit(d[p])) return 0;
        for (; p < end; ++p) {
            const u32 c = d[p];
            if (c == '_') {
                if (p + 1 >= end || !adj_digit(d[p + 1])) return 0;
                continue;
            }
            if (!adj_digit(c)) return 0;
            if (ex < 100000) ex = ex * 10 + (c - '0');
        }
        if (eneg) ex = -ex;
    }
    if (p != end) return 0;
    if (!neg || (nzi < 0 && nzf < 0)) return 1;
    // |w| in [10^(k-1), 10^k): k from the first non-zero digit and the exponent
    const long long k = (nzi >= 0 ? (long long)(ni - nzi) : -(long long)nzf) + ex;
    if (k - 1 >= -300) return 2;
    if (k <= -324) return 1;                     // < 1e-324: rounds to -0.0
    return 3;
}

__global__ void __launch_bounds__(ADJ_THREADS)
k_adj_parse(const uint8_t* __restrict__ d, i64 L, const u64* __restrict__ toff, i64 n, i64 m, int weighted,
            i64* __restrict__ off, int32_t* __restrict__ tgt, unsigned long long* err, unsigned long long* unc,
            unsigned long long* unc_cnt) {
    __shared__ u32 s_w[ADJ_THREADS / 32];
    const i64 b0 = (i64)blockIdx.x * ADJ_TILE + (i64)threadIdx.x * ADJ_BPT;
    u32 mask = b0 < L ? adj_starts(d, L, b0) : 0u;
    const u32 c = __popc(mask);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32 inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[wid] = inc;
    __syncthreads();
    u32 wbase = 0;
    for (int i = 0; i < wid; ++i) wbase += s_w[i];
    u64 t = toff[blockIdx.x] + wbase + inc - c;
    while (mask) {
        const int k = __ffs(mask) - 1;
        mask &= mask - 1;
        const i64 p = b0 + k;
        const u64 tok = t++;
        if (tok < 3) continue;
        const u64 q = tok - 3;
        const i64 end = adj_tok_end(d, L, p);
        if (q < (u64)n) {
            i64 v = 0;
            const int r = adj_parse_int(d, p, end, &v);
            if (r == 0) atomicMin(err + PASGAL_ADJ_INV_OFFSET, (unsigned long long)q);
            else if (r == 2) atomicMin(err + PASGAL_ADJ_OVF_OFFSET, (unsigned long long)q);
            else {
                off[q] = v;
                if (v < 0 || v > m) atomicMin(err + PASGAL_ADJ_RANGE_OFFSET, (unsigned long long)q);
            }
        } else if (q - n < (u64)m) {
            const u64 e = q - n;
            i64 v = 0;
            const int r = adj_parse_int(d, p, end, &v);
            if (r == 0) atomicMin(err + PASGAL_ADJ_INV_TARGET, (unsigned long long)e);
            else if (r == 2) atomicMin(err + PASGAL_ADJ_OVF_TARGET, (unsigned long long)e);
            else if (v < 0 || v >= n) {
                atomicMin(err + PASGAL_ADJ_RANGE_TARGET, (unsigned long long)e);
                tgt[e] = 0;
            } else {
                tgt[e] = (int32_t)v;
            }
        } else if (weighted && q - n - m < (u64)m) {
            const u64 e = q - n - m;
            const int r = adj_weight_class(d, p, end);
            if (r == 0) atomicMin(err + PASGAL_ADJ_INV_WEIGHT, (unsigned long long)e);
            else if (r == 2) atomicMin(err + PASGAL_ADJ_BAD_WEIGHT, (unsigned long long)e);
            else if (r == 3) {
                const unsigned long long s = atomicAdd(unc_cnt, 1ull);
                if (s < PASGAL_ADJ_UNC_CAP) unc[s] = e;
            }
        }
    }
}

// byte position of token k (k >= total: L); one thread: binary search over the tiles'
// exclusive token offsets, then a walk through the tile
__global__ void k_adj_find(const uint8_t* __restrict__ d, i64 L, const u64* __restrict__ toff, i64 ntiles, u64 total,
                           u64 k, long long* out) {
    if (k >= total) {
        out[0] = L;
        return;
    }
    i64 lo = 0, hi = ntiles - 1;   // last tile with toff <= k
    while (lo < hi) {
        const i64 mid = (lo + hi + 1) >> 1;
        if (toff[mid] <= k) lo = mid; else hi = mid - 1;
    }
    u64 t = toff[lo];
    for (i64 b = lo * ADJ_TILE; b < L; b += ADJ_BPT) {
        u32 mask = adj_starts(d, L, b);
        while (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            if (t == k) {
                out[0] = b + j;
                return;
            }
            ++t;
        }
    }
    out[0] = L;
}

// out[1] += number of '\n' in [0, limit)
__global__ void k_adj_count_nl(const uint8_t* __restrict__ d, const long long* limit_p, long long* out) {
    const i64 limit = *limit_p;
    u32 c = 0;
    for (i64 b = ((i64)blockIdx.x * blockDim.x + threadIdx.x) * 16; b < limit; b += (i64)gridDim.x * blockDim.x * 16) {
        for (int k = 0; k < 16 && b + k < limit; ++k) c += d[b + k] == '\n';
    }
    c = __reduce_add_sync(0xFFFFFFFFu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long*)out + 1, (unsigned long long)c);
}

struct AdjTemp {
    u64 *tcnt, *toff, *scan, *total;
    unsigned long long *err, *unc, *unc_cnt;
    long long* pos;
};

static i64 adj_tiles(i64 L) { return L > 0 ? cdiv(L, ADJ_TILE) : 1; }

static size_t adj_carve(AdjTemp& a, char* base, i64 L) {
    size_t o = 0;
    auto take = [&](size_t bytes) -> char* {
        o = (o + 255) & ~(size_t)255;
        char* p = base ? base + o : nullptr;
        o += bytes;
        return p;
    };
    const i64 nt = adj_tiles(L);
    a.tcnt = (u64*)take(8 * nt);
    a.toff = (u64*)take(8 * nt);
    a.scan = (u64*)take(scan_status_bytes(nt));
    a.total = (u64*)take(8);
    a.err = (unsigned long long*)take(8 * PASGAL_ADJ_NERR);
    a.unc = (unsigned long long*)take(8 * PASGAL_ADJ_UNC_CAP);
    a.unc_cnt = (unsigned long long*)take(8);
    a.pos = (long long*)take(16);
    return o + 256;
}

size_t adj_temp_bytes(i64 L) {
    AdjTemp a;
    return adj_carve(a, nullptr, L);
}

int adj_tokenize(const uint8_t* text, i64 L, void* temp, size_t temp_bytes, int64_t* ntokens, cudaStream_t st) {
    AdjTemp a;
    if (temp_bytes < adj_carve(a, nullptr, L)) return PASGAL_EWORKSPACE;
    adj_carve(a, (char*)temp, L);
    const i64 nt = adj_tiles(L);
    if (L > 0) {
        k_adj_count<<<(unsigned)nt, ADJ_THREADS, 0, st>>>(text, L, a.tcnt);
        PG_LAUNCH_CHECK();
        PG_CUDA_TRY(launch_scan<u64>(nt, a.scan, 0ull, SumOp(), AdjLoad{a.tcnt}, AdjStore{a.toff}, a.total, st));
    } else {
        PG_CUDA_TRY(cudaMemsetAsync(a.toff, 0, 8, st));
        PG_CUDA_TRY(cudaMemsetAsync(a.total, 0, 8, st));
    }
    u64 h = 0;
    PG_CUDA_TRY(cudaMemcpyAsync(&h, a.total, 8, cudaMemcpyDeviceToHost, st));
    PG_CUDA_TRY(cudaStreamSynchronize(st));
    *ntokens = (int64_t)h;
    return PASGAL_OK;
}

int adj_token_position(const uint8_t* text, i64 L, void* temp, size_t temp_bytes, i64 k, int64_t* byte_line,
                       cudaStream_t st) {
    AdjTemp a;
    if (temp_bytes < adj_carve(a, nullptr, L)) return PASGAL_EWORKSPACE;
    adj_carve(a, (char*)temp, L);
    u64 total = 0;
    PG_CUDA_TRY(cudaMemcpyAsync(&total, a.total, 8, cudaMemcpyDeviceToHost, st));
    PG_CUDA_TRY(cudaStreamSynchronize(st));
    PG_CUDA_TRY(cudaMemsetAsync(a.pos, 0, 16, st));
    k_adj_find<<<1, 1, 0, st>>>(text, L, a.toff, adj_tiles(L), total, (u64)k, a.pos);
    PG_LAUNCH_CHECK();
    if (L > 0) {
        const i64 blocks = cdiv(L, 256 * 16) < 148 * 16 ? cdiv(L, 256 * 16) : 148 * 16;
        k_adj_count_nl<<<(unsigned)blocks, 256, 0, st>>>(text, a.pos, a.pos);
        PG_LAUNCH_CHECK();
    }
    long long h[2];
    PG_CUDA_TRY(cudaMemcpyAsync(h, a.pos, 16, cudaMemcpyDeviceToHost, st));
    PG_CUDA_TRY(cudaStreamSynchronize(st));
    byte_line[0] = h[0];
    byte_line[1] = h[1] + 1;
    return PASGAL_OK;
}

int adj_parse(const uint8_t* text, i64 L, void* temp, size_t temp_bytes, i64 n, i64 m, int weighted, i64* offsets,
              int32_t* targets, int64_t* first_err, int64_t* uncertain, int64_t* n_uncertain, cudaStream_t st) {
    AdjTemp a;
    if (temp_bytes < adj_carve(a, nullptr, L)) return PASGAL_EWORKSPACE;
    adj_carve(a, (char*)temp, L);
    PG_CUDA_TRY(cudaMemsetAsync(a.err, 0xFF, 8 * PASGAL_ADJ_NERR, st));
    PG_CUDA_TRY(cudaMemsetAsync(a.unc_cnt, 0, 8, st));
    if (L > 0) {
        k_adj_parse<<<(unsigned)adj_tiles(L), ADJ_THREADS, 0, st>>>(text, L, a.toff, n, m, weighted, offsets, targets,
                                                                    a.err, a.unc, a.unc_cnt);
        PG_LAUNCH_CHECK();
    }
    const long long mm = m;
    PG_CUDA_TRY(cudaMemcpyAsync(offsets + n, &mm, 8, cudaMemcpyHostToDevice, st));   // offsets[n] = m
    unsigned long long e[PASGAL_ADJ_NERR], uc = 0;
    PG_CUDA_TRY(cudaMemcpyAsync(e, a.err, sizeof e, cudaMemcpyDeviceToHost, st));
    PG_CUDA_TRY(cudaMemcpyAsync(&uc, a.unc_cnt, 8, cudaMemcpyDeviceToHost, st));
    PG_CUDA_TRY(cudaStreamSynchronize(st));
    const i64 nu = uc < (unsigned long long)PASGAL_ADJ_UNC_CAP ? (i64)uc : PASGAL_ADJ_UNC_CAP;
    if (nu > 0 && uncertain) {
        PG_CUDA_TRY(cudaMemcpyAsync(uncertain, a.unc, 8 * nu, cudaMemcpyDeviceToHost, st));
        PG_CUDA_TRY(cudaStreamSynchronize(st));
    }
    for (int i = 0; i < PASGAL_ADJ_NERR; ++i) first_err[i] = e[i] == ~0ull ? -1 : (int64_t)e[i];
    if (n_uncertain) *n_uncertain = (int64_t)uc;
    return PASGAL_OK;
}

}  // namespace pg
