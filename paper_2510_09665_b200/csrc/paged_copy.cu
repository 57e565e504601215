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

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

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

// ---- unit kernel: the launch as a flat list of <= 4 KiB page pieces ----------
//
// The tile kernel above resolves a tile with one thread (binary search over
// the descriptor prefix, then the page-table reads) while the CTA waits, and
// hands out work in ~64 KiB tiles. Over a whole prompt (80 layers, 5 GiB per
// launch) that is hidden behind the other CTA on the SM; at the launch sizes
// the layerwise connector issues (one layer: 8-64 MiB) it is not: a 64 MiB
// launch measured 0.68 of the HBM peak and an 8 MiB one 0.21-0.25
// (profiles/r02_k12_layers.jsonl), i.e. a ~10 us fixed cost per launch made
// of the serial resolve chains and of 1024 tiles quantised over 296 CTAs.
//
// Here every warp is independent. A unit is (layer, descriptor, page, part):
// at most 4 KiB of one page run, contiguous on both sides. Warp w takes units
// w, w + warps, ...; it finds the descriptor by binary search over the
// one-layer page prefix held in shared memory (loaded once per CTA), reads the
// descriptor and ONE page-table entry, and its 32 lanes move the piece with up
// to 8 x 16-byte loads in flight each. No block-wide barrier after the
// prefix load, no idle threads during a resolve, and 4 KiB granularity keeps
// the tail short. Requires one page per tile (the plan's tile prefix is then
// a page prefix, times n_layers), a contiguous row layout and 16-byte
// alignment; other launches use the tile kernel.
constexpr int kUnitBytes = 4096;
constexpr int kUnitVecs = kUnitBytes / 16 / 32;  // vectors per lane per unit
constexpr uint32_t kSmemDescs = 4096;
constexpr uint64_t kUnitMaxBytes = 512ull << 20;

// Affine plans (PagedCopyPlan::aff_*: one query's consecutive chunks, the
// connector's usual one-layer launch): every address comes from the launch
// parameters, so the page-table entry is the only load in front of the data
// (the general path below adds the descriptor prefix, a block barrier, the
// search and the descriptor itself: ~2 us per launch at 8 MiB,
// tools/microbench_k12_small.cu).
__device__ __forceinline__ void units_affine(const PagedLayout& L, const PagedCopyPlan& P, int dir,
                                             uint32_t parts, uint32_t part_bytes) {
    const uint32_t U = P.aff_pages;
    const uint32_t pages1 = (P.n_desc - 1) * U + (P.aff_last_tokens + L.page_tokens - 1) / L.page_tokens;
    const uint32_t total = pages1 * P.n_layers * parts;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (kThreads / 32);
    const uint32_t w = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    const uint32_t u0 = uint32_t(uint64_t(total) * w / warps);
    const uint32_t u1 = uint32_t(uint64_t(total) * (w + 1) / warps);
    const uint64_t page_run = uint64_t(L.page_tokens) * L.bpt;
    for (uint32_t u = u0; u < u1; ++u) {
        const uint32_t g = u / parts, q = u - g * parts;
        const uint32_t ll = g / pages1, g1 = g - ll * pages1;
        const uint32_t d = g1 / U, j = g1 - d * U;
        const uint32_t layer = P.layer_begin + ll;
        const uint32_t n_tokens = d + 1 == P.n_desc ? P.aff_last_tokens : U * L.page_tokens;
        const uint32_t page_valid = min(L.page_tokens, n_tokens - j * L.page_tokens) * L.bpt;
        const uint32_t begin = q * part_bytes;
        const uint32_t end = min(begin + part_bytes, page_valid);
        if (begin >= end) continue;
        const uint32_t page = uint32_t(__ldg(P.aff_table + uint64_t(L.shared_table ? 0 : layer) * P.aff_table_stride +
                                             P.aff_first_page + g1));
        const uint64_t pbase =
            L.layer_base ? __ldg(reinterpret_cast<const unsigned long long*>(L.layer_base) + layer) : L.base;
        const uint8_t* page_p = reinterpret_cast<const uint8_t*>(pbase + uint64_t(page) * L.page_stride);
        const uint64_t chunk = P.aff_chunk0 + uint64_t(d) * P.aff_chunk_stride + uint64_t(layer) * P.aff_layer_stride +
                               uint64_t(j) * page_run;
        const uint8_t* src = dir == int(CopyDir::gather) ? page_p + begin : reinterpret_cast<const uint8_t*>(chunk + begin);
        uint8_t* dst = dir == int(CopyDir::gather) ? reinterpret_cast<uint8_t*>(chunk + begin)
                                                   : const_cast<uint8_t*>(page_p + begin);
        const uint32_t nv = (end - begin) >> 4;
        int4 v[kUnitVecs];
#pragma unroll
        for (int k = 0; k < kUnitVecs; ++k) {
            const uint32_t i = lane + 32u * k;
            if (i < nv) v[k] = __ldcs(reinterpret_cast<const int4*>(src) + i);
        }
#pragma unroll
        for (int k = 0; k < kUnitVecs; ++k) {
            const uint32_t i = lane + 32u * k;
            if (i < nv) __stcs(reinterpret_cast<int4*>(dst) + i, v[k]);
        }
    }
}

__global__ void __launch_bounds__(kThreads, 2)
paged_copy_units_kernel(const PagedLayout L, const PagedCopyPlan P, const int dir, const uint32_t parts,
                        const uint32_t part_bytes) {
    if (P.aff_pages) {  // (uniform over the launch)
        units_affine(L, P, dir, parts, part_bytes);
        return;
    }
    __shared__ uint32_t s_pb[kSmemDescs + 1];
    const uint32_t nl = P.n_layers;
    const bool smem = P.n_desc <= kSmemDescs;
    if (smem)
        for (uint32_t i = threadIdx.x; i <= P.n_desc; i += kThreads) s_pb[i] = __ldg(P.tile_base + i) / nl;
    __syncthreads();
    auto prefix = [&](uint32_t d) { return smem ? s_pb[d] : __ldg(P.tile_base + d) / nl; };
    const uint32_t pages1 = __ldg(P.tile_base + P.n_desc) / nl;  // pages of one layer over all descriptors
    const uint32_t total = pages1 * nl * parts;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (kThreads / 32);
    const uint32_t w = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    // Warp w owns the contiguous unit range [u0, u1): consecutive units are the
    // parts of one page, then the next page of the same descriptor, so after
    // the first unit the warp resolves by stepping (no search) and re-reads
    // the descriptor / page-table entry from L1.
    const uint32_t u0 = uint32_t(uint64_t(total) * w / warps);
    const uint32_t u1 = uint32_t(uint64_t(total) * (w + 1) / warps);
    if (u0 >= u1) return;
    uint32_t g = u0 / parts;
    uint32_t q = u0 - g * parts;
    uint32_t ll = g / pages1;
    uint32_t g1 = g - ll * pages1;
    uint32_t lo = 0, hi = P.n_desc;  // largest d with prefix[d] <= g1
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (prefix(mid) <= g1) lo = mid; else hi = mid;
    }
    uint32_t next_base = prefix(lo + 1);  // first page of descriptor lo + 1
    const uint8_t* page_p = nullptr;
    uint64_t chunk = 0;
    uint32_t page_valid = 0;  // bytes of the current page run
    bool fresh = true;        // page addresses need resolving
    for (uint32_t u = u0; u < u1; ++u) {
        if (fresh) {
            const XferDesc* dp = P.descs + lo;
            const uint32_t j = g1 - prefix(lo);
            const uint32_t n_tokens = __ldg(&dp->n_tokens);
            page_valid = min(L.page_tokens, n_tokens - j * L.page_tokens) * L.bpt;
            const uint32_t layer = P.layer_begin + ll;
            const int32_t* table =
                reinterpret_cast<const int32_t*>(__ldg(reinterpret_cast<const unsigned long long*>(&dp->table)));
            const uint32_t page = uint32_t(__ldg(table + uint64_t(L.shared_table ? 0 : layer) * __ldg(&dp->table_stride) +
                                                 __ldg(&dp->first_page) + j));
            const uint64_t pbase =
                L.layer_base ? __ldg(reinterpret_cast<const unsigned long long*>(L.layer_base) + layer) : L.base;
            page_p = reinterpret_cast<const uint8_t*>(pbase + uint64_t(page) * L.page_stride);
            chunk = __ldg(reinterpret_cast<const unsigned long long*>(&dp->chunk)) +
                    uint64_t(layer) * __ldg(reinterpret_cast<const unsigned long long*>(&dp->layer_stride)) +
                    uint64_t(j) * L.page_tokens * L.bpt;
            fresh = false;
        }
        const uint32_t begin = q * part_bytes;
        const uint32_t end = min(begin + part_bytes, page_valid);
        if (begin < end) {  // (empty: a part past the short last page of a descriptor)
            const uint8_t* src = dir == int(CopyDir::gather) ? page_p + begin
                                                             : reinterpret_cast<const uint8_t*>(chunk + begin);
            uint8_t* dst = dir == int(CopyDir::gather) ? reinterpret_cast<uint8_t*>(chunk + begin)
                                                       : const_cast<uint8_t*>(page_p + begin);
            const uint32_t nv = (end - begin) >> 4;
            int4 v[kUnitVecs];
#pragma unroll
            for (int k = 0; k < kUnitVecs; ++k) {
                const uint32_t i = lane + 32u * k;
                if (i < nv) v[k] = __ldcs(reinterpret_cast<const int4*>(src) + i);
            }
#pragma unroll
            for (int k = 0; k < kUnitVecs; ++k) {
                const uint32_t i = lane + 32u * k;
                if (i < nv) __stcs(reinterpret_cast<int4*>(dst) + i, v[k]);
            }
        }
        // step to unit u + 1
        if (++q == parts) {
            q = 0;
            fresh = true;
            if (++g1 == pages1) {  // next layer: descriptors from the start
                g1 = 0;
                ++ll;
                lo = 0;
                next_base = prefix(1);
            }
            while (g1 >= next_base) next_base = prefix(++lo + 1);
        }
    }
}

// ---- bulk-copy (TMA) variant of the unit kernel ------------------------------
//
// Same units and per-warp ranges as paged_copy_units_kernel, but the bytes
// move through the copy engine of the SM (cp.async.bulk): lane 0 of each warp
// keeps kBulkStages units in flight — a bulk load global -> shared (completion
// on an mbarrier with the byte count), then a bulk store shared -> global —
// and no thread touches the data. Selected with TKV_PAGED_KERNEL=bulk (A/B,
// profiles/r02_k12_layers_bulk.jsonl); the LSU version is the default.
constexpr int kBulkWarps = 4;
constexpr int kBulkStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(32 * kBulkWarps)
paged_copy_bulk_kernel(const PagedLayout L, const PagedCopyPlan P, const int dir, const uint32_t parts,
                       const uint32_t part_bytes) {
    extern __shared__ __align__(128) uint8_t bulk_smem[];
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane != 0) return;  // one issuing thread per warp; the SM's bulk-copy unit moves the bytes
    uint8_t* buf = bulk_smem + size_t(wid) * kBulkStages * kUnitBytes;
    __shared__ __align__(8) unsigned long long bars[kBulkWarps][kBulkStages];
    for (int st = 0; st < kBulkStages; ++st)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[wid][st])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

    const uint32_t nl = P.n_layers;
    auto prefix = [&](uint32_t d) { return __ldg(P.tile_base + d) / nl; };
    const uint32_t pages1 = __ldg(P.tile_base + P.n_desc) / nl;
    const uint32_t total = pages1 * nl * parts;
    const uint32_t warps = gridDim.x * kBulkWarps;
    const uint32_t w = blockIdx.x * kBulkWarps + wid;
    const uint32_t u0 = uint32_t(uint64_t(total) * w / warps);
    const uint32_t u1 = uint32_t(uint64_t(total) * (w + 1) / warps);
    if (u0 >= u1) return;
    // unit -> (src, dst, bytes), stepping like the unit kernel
    uint32_t g = u0 / parts, q = u0 - (u0 / parts) * parts;
    uint32_t ll = g / pages1, g1 = g - ll * pages1;
    uint32_t lo = 0, hi = P.n_desc;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (prefix(mid) <= g1) lo = mid; else hi = mid;
    }
    uint32_t next_base = prefix(lo + 1);
    const uint8_t* page_p = nullptr;
    uint64_t chunk = 0;
    uint32_t page_valid = 0;
    bool fresh = true;
    auto next = [&](const uint8_t*& src, uint8_t*& dst, uint32_t& bytes) {
        for (;;) {
            if (fresh) {
                const XferDesc* dp = P.descs + lo;
                const uint32_t j = g1 - prefix(lo);
                page_valid = min(L.page_tokens, __ldg(&dp->n_tokens) - j * L.page_tokens) * L.bpt;
                const uint32_t layer = P.layer_begin + ll;
                const int32_t* table = reinterpret_cast<const int32_t*>(
                    __ldg(reinterpret_cast<const unsigned long long*>(&dp->table)));
                const uint32_t page = uint32_t(__ldg(table + uint64_t(L.shared_table ? 0 : layer) * __ldg(&dp->table_stride) +
                                                     __ldg(&dp->first_page) + j));
                const uint64_t pbase =
                    L.layer_base ? __ldg(reinterpret_cast<const unsigned long long*>(L.layer_base) + layer) : L.base;
                page_p = reinterpret_cast<const uint8_t*>(pbase + uint64_t(page) * L.page_stride);
                chunk = __ldg(reinterpret_cast<const unsigned long long*>(&dp->chunk)) +
                        uint64_t(layer) * __ldg(reinterpret_cast<const unsigned long long*>(&dp->layer_stride)) +
                        uint64_t(j) * L.page_tokens * L.bpt;
                fresh = false;
            }
            const uint32_t begin = q * part_bytes;
            const uint32_t end = min(begin + part_bytes, page_valid);
            const bool have = begin < end;
            if (have) {
                src = dir == int(CopyDir::gather) ? page_p + begin : reinterpret_cast<const uint8_t*>(chunk + begin);
                dst = dir == int(CopyDir::gather) ? reinterpret_cast<uint8_t*>(chunk + begin)
                                                  : const_cast<uint8_t*>(page_p + begin);
                bytes = end - begin;
            }
            if (++q == parts) {
                q = 0;
                fresh = true;
                if (++g1 == pages1) {
                    g1 = 0;
                    ++ll;
                    lo = 0;
                    next_base = ll < nl ? prefix(1) : 0;
                }
                while (ll < nl && g1 >= next_base) next_base = prefix(++lo + 1);
            }
            if (have) return true;
            if (ll >= nl) return false;
        }
    };
    uint32_t limit = u1 - u0;  // units of this warp (a trailing empty part ends it early)
    uint8_t* dsts[kBulkStages];
    uint32_t sizes[kBulkStages];
    uint32_t issued = 0;
    auto issue_load = [&](uint32_t i) -> bool {
        const uint8_t* src;
        uint8_t* dst;
        uint32_t bytes;
        if (!next(src, dst, bytes)) return false;
        const int st = int(i % kBulkStages);
        dsts[st] = dst;
        sizes[st] = bytes;
        const uint32_t bar = smem_u32(&bars[wid][st]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(buf + size_t(st) * kUnitBytes)),
                     "l"(src), "r"(bytes), "r"(bar)
                     : "memory");
        return true;
    };
    // prologue: up to kBulkStages loads in flight
    while (issued < kBulkStages && issued < limit) {
        if (!issue_load(issued)) {
            limit = issued;
            break;
        }
        ++issued;
    }
    for (uint32_t done = 0; done < issued; ++done) {
        const int st = int(done % kBulkStages);
        const uint32_t phase = (done / kBulkStages) & 1;
        const uint32_t bar = smem_u32(&bars[wid][st]);
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dsts[st]),
                     "r"(smem_u32(buf + size_t(st) * kUnitBytes)), "r"(sizes[st])
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (issued < limit) {
            // the stage is reused once its store has read it
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            if (issue_load(issued))
                ++issued;
            else
                limit = issued;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int W, bool CONTIG>
cudaError_t launch_w(const PagedLayout& L, const PagedCopyPlan& P, CopyDir dir, int ctas,
                     cudaStream_t s) {
    constexpr int U = W >= 8 ? 4 : 8;
    if (uint32_t(ctas) > P.total_tiles) ctas = int(P.total_tiles);
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

namespace {
// TKV_PAGED_AFFINE=0: plans built in affine form take the general unit-kernel
// path anyway (A/B measurements only).
bool affine_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("TKV_PAGED_AFFINE");
        return !(v && std::strcmp(v, "0") == 0);
    }();
    return on;
}

// 4 KiB pieces of a page run (the unit kernel's units)
void unit_parts(uint64_t page_bytes, uint32_t& parts, uint32_t& part_bytes) {
    parts = uint32_t((page_bytes + kUnitBytes - 1) / kUnitBytes);
    part_bytes = uint32_t(((page_bytes + parts - 1) / parts + 15) & ~uint64_t(15));
}
}  // namespace

cudaError_t launch_paged_copy_affine(const PagedLayout& L, const PagedCopyPlan& P, CopyDir dir, int ctas,
                                     cudaStream_t stream) {
    if (P.aff_pages == 0 || P.n_desc == 0 || P.n_layers == 0) return cudaSuccess;
    const uint64_t a = L.bpt | L.page_stride | L.base | P.aff_chunk0 | P.aff_chunk_stride | P.aff_layer_stride;
    if ((a & 15) || L.n_planes != 1 || L.token_stride != L.bpt || L.page_tokens == 0) return cudaErrorInvalidValue;
    if (P.aff_last_tokens == 0 || P.aff_last_tokens > P.aff_pages * L.page_tokens) return cudaErrorInvalidValue;
    const uint64_t page_bytes = uint64_t(L.page_tokens) * L.bpt;
    uint32_t parts, part_bytes;
    unit_parts(page_bytes, parts, part_bytes);
    const uint64_t pages1 =
        uint64_t(P.n_desc - 1) * P.aff_pages + (P.aff_last_tokens + L.page_tokens - 1) / L.page_tokens;
    const uint64_t units = pages1 * P.n_layers * parts;
    if (units >= (1ull << 32)) return cudaErrorInvalidValue;
    if (ctas <= 0) ctas = 2 * sm_count();
    const uint64_t want = (units + kThreads / 32 - 1) / (kThreads / 32);
    if (uint64_t(ctas) > want) ctas = int(want);
    note_launch();
    paged_copy_units_kernel<<<ctas, kThreads, 0, stream>>>(L, P, int(dir), parts, part_bytes);
    return cudaGetLastError();
}

cudaError_t launch_paged_copy(const PagedLayout& L, const PagedCopyPlan& Pin, CopyDir dir, int ctas,
                              cudaStream_t stream) {
    PagedCopyPlan P = Pin;
    if (!affine_enabled()) P.aff_pages = 0;
    if (P.total_tiles == 0 || P.n_desc == 0) return cudaSuccess;
    if (P.pages_per_tile == 0 || P.pages_per_tile > kMaxPagesPerTile) return cudaErrorInvalidValue;
    if (ctas <= 0) ctas = 2 * sm_count();
    // Vector width: the largest of 16/8/4/1 dividing every stride and base.
    uint64_t a = L.bpt | L.plane_bytes | L.token_stride | L.page_stride | L.plane_stride | L.base |
                 P.addr_or;
    const bool contig = L.n_planes == 1 && L.token_stride == L.bpt;
    const uint64_t page_bytes = uint64_t(L.page_tokens) * L.bpt;
    // TKV_PAGED_KERNEL=tile forces the tile kernel (A/B measurements only).
    static const bool force_tile = [] {
        const char* v = std::getenv("TKV_PAGED_KERNEL");
        return v != nullptr && std::strcmp(v, "tile") == 0;
    }();
    static const bool use_bulk = [] {
        const char* v = std::getenv("TKV_PAGED_KERNEL");
        return v != nullptr && std::strcmp(v, "bulk") == 0;
    }();
    // Unit kernel for launches up to kUnitMaxBytes (one layer of a batch);
    // bigger ones (all layers at once) keep the tile kernel, whose sweep over
    // consecutive tiles measured faster at that size (1.04 vs 0.95 of peak
    // at 5 GiB, profiles/r02_k12_layers.jsonl).
    const uint64_t launch_bytes = uint64_t(P.total_tiles) * page_bytes;
    if ((a & 15) == 0 && contig && P.pages_per_tile == 1 && launch_bytes <= kUnitMaxBytes && !force_tile) {
        uint32_t parts, part_bytes;
        unit_parts(page_bytes, parts, part_bytes);
        if (uint64_t(P.total_tiles) * parts < (1ull << 32)) {
            const uint64_t units = uint64_t(P.total_tiles) * parts;
            const uint64_t want = (units + kThreads / 32 - 1) / (kThreads / 32);  // at least one unit per warp
            if (uint64_t(ctas) > want) ctas = int(want);
            note_launch();
            if (use_bulk) {
                const size_t smem = size_t(kBulkWarps) * kBulkStages * kUnitBytes;
                static const cudaError_t attr = cudaFuncSetAttribute(
                    paged_copy_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
                if (attr != cudaSuccess) return attr;
                const uint64_t bwant = (units + kBulkWarps - 1) / kBulkWarps;
                const int bctas = int(std::min<uint64_t>(bwant, uint64_t(3 * sm_count())));
                paged_copy_bulk_kernel<<<bctas, 32 * kBulkWarps, smem, stream>>>(L, P, int(dir), parts, part_bytes);
                return cudaGetLastError();
            }
            paged_copy_units_kernel<<<ctas, kThreads, 0, stream>>>(L, P, int(dir), parts, part_bytes);
            return cudaGetLastError();
        }
    }
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
