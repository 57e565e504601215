// Small one-layer paged copies (the layerwise connector's K1 / K2 launch
// sizes): what the indirection costs against a plain contiguous copy of the
// same bytes. Per variant: back-to-back launches timed with CUDA events
// (steady-state cost per launch) and one launch alone (event pair around it).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_k12 tools/microbench_k12_small.cu && /tmp/mb_k12
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

constexpr int kThreads = 512;
constexpr int kMaxParamPages = 4096;

__global__ void empty_kernel() {}

// warp w copies bytes [w*4K, (w+1)*4K): 32 lanes x 8 x 16 B
__global__ void __launch_bounds__(kThreads) contig_kernel(const int4* __restrict__ src, int4* __restrict__ dst,
                                                          uint32_t units) {
    const uint32_t w = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    for (uint32_t u = w; u < units; u += gridDim.x * (kThreads / 32)) {
        const int4* s = src + uint64_t(u) * 256;
        int4* d = dst + uint64_t(u) * 256;
        int4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldcs(s + lane + 32 * k);
#pragma unroll
        for (int k = 0; k < 8; ++k) __stcs(d + lane + 32 * k, v[k]);
    }
}

// gather: unit u = (page j = u / parts, part q): page id from a device table (one dependent load)
__global__ void __launch_bounds__(kThreads) table_kernel(const uint8_t* __restrict__ pool, const int32_t* __restrict__ table,
                                                         uint8_t* __restrict__ chunk, uint32_t units, uint32_t parts,
                                                         uint32_t page_bytes) {
    const uint32_t w = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    for (uint32_t u = w; u < units; u += gridDim.x * (kThreads / 32)) {
        const uint32_t j = u / parts, q = u - j * parts;
        const int32_t page = __ldg(table + j);
        const int4* s = reinterpret_cast<const int4*>(pool + uint64_t(page) * page_bytes + q * 4096);
        int4* d = reinterpret_cast<int4*>(chunk + uint64_t(j) * page_bytes + q * 4096);
        int4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldcs(s + lane + 32 * k);
#pragma unroll
        for (int k = 0; k < 8; ++k) __stcs(d + lane + 32 * k, v[k]);
    }
}

struct ParamPages {
    int32_t page[kMaxParamPages];
};
// same, page ids in the kernel's parameter space (constant bank): no dependent global load
__global__ void __launch_bounds__(kThreads) param_kernel(const uint8_t* __restrict__ pool, const __grid_constant__ ParamPages P,
                                                         uint8_t* __restrict__ chunk, uint32_t units, uint32_t parts,
                                                         uint32_t page_bytes) {
    const uint32_t w = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    for (uint32_t u = w; u < units; u += gridDim.x * (kThreads / 32)) {
        const uint32_t j = u / parts, q = u - j * parts;
        const int32_t page = P.page[j];
        const int4* s = reinterpret_cast<const int4*>(pool + uint64_t(page) * page_bytes + q * 4096);
        int4* d = reinterpret_cast<int4*>(chunk + uint64_t(j) * page_bytes + q * 4096);
        int4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldcs(s + lane + 32 * k);
#pragma unroll
        for (int k = 0; k < 8; ++k) __stcs(d + lane + 32 * k, v[k]);
    }
}

template <typename F>
void timeit(const char* name, double bytes, F launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 5; ++i) launch(i);
    cudaDeviceSynchronize();
    const int n = 80;
    cudaEventRecord(a);
    for (int i = 0; i < n; ++i) launch(i);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double us_b2b = 1e3 * ms / n;
    std::vector<float> one;
    for (int i = 0; i < 20; ++i) {
        cudaEventRecord(a);
        launch(i);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        one.push_back(1e3f * ms);
    }
    std::sort(one.begin(), one.end());
    printf("{\"variant\": \"%s\", \"bytes\": %.0f, \"us_back_to_back\": %.2f, \"us_alone_median\": %.2f, \"gbs_b2b\": %.0f}\n",
           name, bytes, us_b2b, one[10], bytes > 0 ? 2 * bytes / us_b2b / 1e3 : 0.0);
}

int main() {
    for (uint32_t page_bytes : {16u * 512u, 16u * 4096u}) {  // bpt 512 (TP=8) and 4096 (TP=1)
        const uint32_t pages = 1024;                           // 16K tokens of one layer
        const uint64_t bytes = uint64_t(pages) * page_bytes;
        const uint32_t parts = page_bytes / 4096, units = pages * parts;
        const uint64_t pool_pages = 80ull * pages;  // a pool of 80 layers: pages spread like the product's
        uint8_t *pool, *chunk;
        int32_t* table;
        cudaMalloc(&pool, pool_pages * page_bytes);
        // 80 distinct chunk-side buffers so nothing is L2-resident between launches
        cudaMalloc(&chunk, 80 * bytes);
        cudaMalloc(&table, 80 * pages * 4);
        std::vector<int32_t> ids(pool_pages);
        std::iota(ids.begin(), ids.end(), 0);
        std::shuffle(ids.begin(), ids.end(), std::mt19937(7));
        cudaMemcpy(table, ids.data(), 80 * pages * 4, cudaMemcpyHostToDevice);
        cudaMemset(pool, 1, pool_pages * page_bytes);
        std::vector<ParamPages> pp(80);
        for (int l = 0; l < 80; ++l)
            for (uint32_t j = 0; j < pages; ++j) pp[l].page[j] = ids[l * pages + j];
        const int grids[] = {148, 296, int((units + 15) / 16)};
        printf("# page_bytes %u, one layer = %.1f MiB\n", page_bytes, bytes / 1048576.0);
        timeit("empty", 0, [&](int) { empty_kernel<<<1, 32>>>(); });
        for (int g : grids) {
            char nm[96];
            snprintf(nm, sizeof nm, "contiguous g=%d", g);
            timeit(nm, bytes, [&](int i) {
                contig_kernel<<<g, kThreads>>>(reinterpret_cast<const int4*>(pool + (i % 80) * bytes),
                                               reinterpret_cast<int4*>(chunk + (i % 80) * bytes), units);
            });
            snprintf(nm, sizeof nm, "paged, device table g=%d", g);
            timeit(nm, bytes, [&](int i) {
                table_kernel<<<g, kThreads>>>(pool, table + (i % 80) * pages, chunk + (i % 80) * bytes, units, parts,
                                              page_bytes);
            });
            snprintf(nm, sizeof nm, "paged, ids in params g=%d", g);
            timeit(nm, bytes, [&](int i) {
                param_kernel<<<g, kThreads>>>(pool, pp[i % 80], chunk + (i % 80) * bytes, units, parts, page_bytes);
            });
        }
        cudaFree(pool);
        cudaFree(chunk);
        cudaFree(table);
    }
    return 0;
}
