// K1 / K2 — multi-layer paged KV gather (store) and scatter (retrieve).
//
// Replaces the reference's per-(layer, chunk) memcpy loops
// PagedKVStore::gather_tokens_into (src/paged_store.cpp:123-140) and
// PagedKVStore::scatter_tokens (src/paged_store.cpp:147-175), as driven by
// Connector::start_store_kv (src/connector.cpp:281-358) and
// Connector::run_load_layer (src/connector.cpp:179-219).
//
// Work decomposition: a "tile" is (chunk descriptor, layer, run of up to
// pages_per_tile pages) — about 64 KiB of payload, contiguous on the chunk
// side ([L][T][bpt] layer-major, kv_chunk.hpp:12-36) and contiguous per page
// on the paged side. A persistent grid walks tiles in order (consecutive CTAs
// stream consecutive tiles); thread 0 resolves the tile (binary search over
// the per-descriptor tile prefix, page-table reads) into shared memory, then
// all threads move 16-byte vectors with UNROLL loads in flight before the
// stores. The chunk side can be HBM, mapped pinned host memory (the
// zero-copy host tier) or a peer GPU's memory: the kernel only sees a
// device-visible address.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace tkv {
namespace {

constexpr int kThreads = 512;
constexpr int kMaxPagesPerTile = 64;

template <int W>
struct Vec;
template <>
struct Vec<16> {
    using T = int4;
};
template <>
struct Vec<8> {
    using T = int2;
};
template <>
struct Vec<4> {
    using T = int;
};
template <>
struct Vec<1> {
    using T = unsigned char;
};

template <int W>
__device__ __forceinline__ typename Vec<W>::T ld_stream(const void* p) {
    using T = typename Vec<W>::T;
    if constexpr (W == 1) {
        return *static_cast<const volatile T*>(p);
    } else {
        return __ldcs(static_cast<const T*>(p));
    }
}

template <int W>
__device__ __forceinline__ void st_stream(void* p, typename Vec<W>::T v) {
    using T = typename Vec<W>::T;
    if constexpr (W == 1) {
        *static_cast<T*>(p) = v;
    } else {
        __stcs(static_cast<T*>(p), v);
    }
}

struct TileInfo {
    uint64_t chunk;       // chunk-side address of the tile's first byte
    uint32_t rows;        // rows in this tile
    uint32_t pages;       // pages in this tile
    uint64_t page_addr[kMaxPagesPerTile];
};

// Resolves tile -> (descriptor, layer, pages) into shared memory.
__device__ void resolve_tile(const PagedLayout& L, const PagedCopyPlan& P, uint32_t tile,
                             TileInfo& ti) {
    // upper_bound over tile_base[0..n_desc] — largest d with tile_base[d] <= tile
    uint32_t lo = 0, hi = P.n_desc;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (P.tile_base[mid] <= tile) lo = mid; else hi = mid;
    }
    const XferDesc d = P.descs[lo];
    const uint32_t local = tile - P.tile_base[lo];
    const uint32_t pages_d = (d.n_tokens + L.page_tokens - 1) / L.page_tokens;
    const uint32_t tiles_per_layer = (pages_d + P.pages_per_tile - 1) / P.pages_per_tile;
    const uint32_t layer = P.layer_begin + local / tiles_per_layer;
    const uint32_t page0 = (local % tiles_per_layer) * P.pages_per_tile;
    const uint32_t pages = min(P.pages_per_tile, pages_d - page0);
    const uint32_t row0 = page0 * L.page_tokens;
    ti.rows = min(pages * L.page_tokens, d.n_tokens - row0);
    ti.pages = pages;
    ti.chunk = d.chunk + uint64_t(layer) * d.layer_stride + uint64_t(row0) * L.bpt;
    const int32_t* row = d.table + uint64_t(L.shared_table ? 0 : layer) * d.table_stride +
                         d.first_page + page0;
    const uint64_t base = L.layer_base ? L.layer_base[layer] : L.base;
    for (uint32_t j = 0; j < pages; ++j) ti.page_addr[j] = base + uint64_t(uint32_t(row[j])) * L.page_stride;
}

// CONTIG: one plane and token_stride == bpt, so each page's rows are one
// contiguous run and the tile is a concatenation of page runs.
template <int W, bool CONTIG, int UNROLL>
__global__ void __launch_bounds__(kThreads, 2)
paged_copy_kernel(const PagedLayout L, const PagedCopyPlan P, const int dir) {
    using T = typename Vec<W>::T;
    __shared__ TileInfo ti;
    const uint32_t page_vecs = L.page_tokens * L.bpt / W;  // vectors in a full page run
    const bool pv_pow2 = (page_vecs & (page_vecs - 1)) == 0;
    const uint32_t pv_shift = pv_pow2 ? __ffs(page_vecs) - 1 : 0;
    const uint32_t pvr = L.plane_bytes / W;                 // vectors per plane-row
    const uint32_t vrow = L.n_planes * pvr;                 // vectors per chunk row

    for (uint32_t tile = blockIdx.x; tile < P.total_tiles; tile += gridDim.x) {
        __syncthreads();  // previous tile fully consumed ti
        if (threadIdx.x == 0) resolve_tile(L, P, tile, ti);
        __syncthreads();
        const uint32_t n = CONTIG ? ti.rows * (L.bpt / W) : ti.rows * vrow;
        uint8_t* const chunk = reinterpret_cast<uint8_t*>(ti.chunk);

        for (uint32_t base = threadIdx.x; base < n; base += kThreads * UNROLL) {
            T v[UNROLL];
            uint8_t* pp[UNROLL];
            uint8_t* cp[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint32_t e = base + u * kThreads;
                const uint32_t ec = e < n ? e : 0;
                if constexpr (CONTIG) {
                    const uint32_t j = pv_pow2 ? (ec >> pv_shift) : (ec / page_vecs);
                    const uint32_t in = ec - j * page_vecs;
                    pp[u] = reinterpret_cast<uint8_t*>(ti.page_addr[j]) + uint64_t(in) * W;
                    cp[u] = chunk + uint64_t(ec) * W;
                } else {
                    const uint32_t r = ec / vrow;
                    const uint32_t rem = ec - r * vrow;
                    const uint32_t q = rem / pvr;
                    const uint32_t c = rem - q * pvr;
                    const uint32_t j = r / L.page_tokens;
                    const uint32_t rr = r - j * L.page_tokens;
                    pp[u] = reinterpret_cast<uint8_t*>(ti.page_addr[j]) + q * L.plane_stride +
                            uint64_t(rr) * L.token_stride + uint64_t(c) * W;
                    cp[u] = chunk + uint64_t(r) * L.bpt + uint64_t(q) * L.plane_bytes +
                            uint64_t(c) * W;
                }
            }
            if (dir == int(CopyDir::gather)) {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u)
                    if (base + u * kThreads < n) v[u] = ld_stream<W>(pp[u]);
#pragma unroll
                for (int u = 0; u < UNROLL; ++u)
                    if (base + u * kThreads < n) st_stream<W>(cp[u], v[u]);
            } else {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u)
                    if (base + u * kThreads < n) v[u] = ld_stream<W>(cp[u]);
#pragma unroll
                for (int u = 0; u < UNROLL; ++u)
                    if (base + u * kThreads < n) st_stream<W>(pp[u], v[u]);
            }
        }
    }
}

template <int W, bool CONTIG>
cudaError_t launch_w(const PagedLayout& L, const PagedCopyPlan& P, CopyDir dir, int ctas,
                     cudaStream_t s) {
    constexpr int U = W >= 8 ? 4 : 8;
    note_launch();
    paged_copy_kernel<W, CONTIG, U><<<ctas, kThreads, 0, s>>>(L, P, int(dir));
    return cudaGetLastError();
}

int sm_count() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

}  // namespace

cudaError_t launch_paged_copy(const PagedLayout& L, const PagedCopyPlan& P, CopyDir dir, int ctas,
                              cudaStream_t stream) {
    if (P.total_tiles == 0 || P.n_desc == 0) return cudaSuccess;
    if (P.pages_per_tile == 0 || P.pages_per_tile > kMaxPagesPerTile) return cudaErrorInvalidValue;
    if (ctas <= 0) ctas = 2 * sm_count();
    if (uint32_t(ctas) > P.total_tiles) ctas = int(P.total_tiles);
    // Vector width: the largest of 16/8/4/1 dividing every stride and base.
    uint64_t a = L.bpt | L.plane_bytes | L.token_stride | L.page_stride | L.plane_stride | L.base |
                 P.addr_or;
    const bool contig = L.n_planes == 1 && L.token_stride == L.bpt;
    if ((a & 15) == 0) return contig ? launch_w<16, true>(L, P, dir, ctas, stream)
                                     : launch_w<16, false>(L, P, dir, ctas, stream);
    if ((a & 7) == 0) return contig ? launch_w<8, true>(L, P, dir, ctas, stream)
                                    : launch_w<8, false>(L, P, dir, ctas, stream);
    if ((a & 3) == 0) return contig ? launch_w<4, true>(L, P, dir, ctas, stream)
                                    : launch_w<4, false>(L, P, dir, ctas, stream);
    return contig ? launch_w<1, true>(L, P, dir, ctas, stream)
                  : launch_w<1, false>(L, P, dir, ctas, stream);
}

}  // namespace tkv
