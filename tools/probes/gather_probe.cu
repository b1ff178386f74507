// Random 4-byte gathers into a large array: time and (under ncu) L2/DRAM sectors per
// gather for different load flavours.  Experiment only (not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int MODE>
__device__ __forceinline__ uint32_t ld(const uint32_t* p) {
    uint32_t r;
    if (MODE == 0) r = __ldg(p);
    else if (MODE == 1) r = __ldcg(p);
    else if (MODE == 2) asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    else if (MODE == 3) r = *(volatile const uint32_t*)p;
    else if (MODE == 4) r = __ldcs(p);
    else if (MODE == 5) asm volatile("ld.global.relaxed.gpu.u32 %0, [%1];" : "=r"(r) : "l"(p));
    else if (MODE == 6) asm volatile("atom.global.or.b32 %0, [%1], 0;" : "=r"(r) : "l"(p));
    else if (MODE == 7) asm volatile("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(r) : "l"(p));
    else asm volatile("ld.global.nc.L1::evict_first.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

template <int MODE, int U>
__global__ void k_gather(const uint32_t* __restrict__ a, uint64_t mask, uint64_t n_items, uint32_t* out) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (uint64_t b = i; b * U < n_items; b += stride) {
        uint32_t v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) v[k] = ld<MODE>(a + (mix(b * U + k) & mask));
#pragma unroll
        for (int k = 0; k < U; ++k) acc += v[k];
    }
    out[i] = acc;
}

template <int MODE>
float run(const uint32_t* a, uint64_t mask, uint64_t items, uint32_t* out, int blocks) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_gather<MODE, 8><<<blocks, 256>>>(a, mask, items, out);
    cudaEventRecord(e0);
    k_gather<MODE, 8><<<blocks, 256>>>(a, mask, items, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

// cp.async 4-byte gathers into shared memory, 8 per thread in flight
__global__ void k_gather_async(const uint32_t* __restrict__ a, uint64_t mask, uint64_t n_items, uint32_t* out) {
    __shared__ uint32_t sb[256 * 8];
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (uint64_t b = i; b * 8 < n_items; b += stride) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint32_t d = (uint32_t)__cvta_generic_to_shared(sb + k * 256 + threadIdx.x);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(a + (mix(b * 8 + k) & mask)) : "memory");
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += sb[k * 256 + threadIdx.x];
    }
    out[i] = acc;
}
float run_async(const uint32_t* a, uint64_t mask, uint64_t items, uint32_t* out, int blocks) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_gather_async<<<blocks, 256>>>(a, mask, items, out);
    cudaEventRecord(e0);
    k_gather_async<<<blocks, 256>>>(a, mask, items, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main(int argc, char** argv) {
    const uint64_t n = 1ull << 28;   // 1 GB of u32
    const uint64_t items = 1ull << 30;
    uint32_t *a, *out;
    cudaMalloc(&a, n * 4);
    cudaMemset(a, 1, n * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8;
    cudaMalloc(&out, (size_t)blocks * 256 * 4);
    const char* names[] = {"ldg", "ldcg", "nc_noalloc", "volatile", "ldcs", "relaxed", "atom_or0", "nc_L2_64B", "L1_evfirst", "cp_async4"};
    for (uint64_t lb : {28ull, 24ull, 22ull}) {   // array span 1 GB, 64 MB, 16 MB
        uint64_t mask = (1ull << lb) - 1;
        float t[10];
        t[0] = run<0>(a, mask, items, out, blocks);
        t[1] = run<1>(a, mask, items, out, blocks);
        t[2] = run<2>(a, mask, items, out, blocks);
        t[3] = run<3>(a, mask, items, out, blocks);
        t[4] = run<4>(a, mask, items, out, blocks);
        t[5] = run<5>(a, mask, items, out, blocks);
        t[6] = run<6>(a, mask, items, out, blocks);
        t[7] = run<7>(a, mask, items, out, blocks);
        t[8] = run<8>(a, mask, items, out, blocks);
        t[9] = run_async(a, mask, items, out, blocks);
        for (int k = 0; k < 10; ++k)
            printf("span 2^%llu u32  %-11s %8.3f ms  %6.2f G gathers/s\n", (unsigned long long)lb, names[k], t[k],
                   items / (t[k] * 1e6));
    }
    if (argc > 1) {   // the L2 fetch-granularity limit, then ldg again
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32);
        size_t g = 0;
        cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
        float t0 = run<0>(a, (1ull << 28) - 1, items, out, blocks);
        printf("limit %zu: ldg span 2^28 %8.3f ms\n", g, t0);
    }
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
