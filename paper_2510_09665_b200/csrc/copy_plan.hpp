// Host-built K1/K2 launch plans shared by the connector and the PD path:
// descriptor variants (one per staging ring slot, or one for direct slot /
// peer access) and tile prefixes for one-layer and all-layer launches,
// uploaded once per batch with a single H2D copy from a pooled pinned block
// (no allocation on the transfer path once the pool is warm).
#pragma once

#include <cstring>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"

namespace tkv {

// Pages per tile of the tile kernel: ~64 KiB tiles.
inline uint32_t pages_per_tile(size_t page_bytes) {
    size_t p = 65536 / (page_bytes ? page_bytes : 1);
    return uint32_t(p < 1 ? 1 : (p > 64 ? 64 : p));
}

inline std::vector<uint32_t> tile_prefix(const std::vector<XferDesc>& d, uint32_t page_tokens,
                                         uint32_t ppt, uint32_t n_layers) {
    std::vector<uint32_t> tb(d.size() + 1, 0);
    for (size_t i = 0; i < d.size(); ++i)
        tb[i + 1] = tb[i] + tiles_for(d[i].n_tokens, page_tokens, ppt, n_layers);
    return tb;
}

// One-layer launches (the layerwise connector: 8-64 MiB each) use one page
// per tile when rows are 16-byte multiples, so they can run the unit kernel
// (paged_copy.cu); all-layer launches keep the tile kernel's ~64 KiB tiles.
inline uint32_t pages_per_tile_one_layer(size_t page_bytes) {
    return page_bytes % 256 == 0 ? 1u : pages_per_tile(page_bytes);
}

// The affine form of a descriptor list (PagedCopyPlan::aff_*), if it has one:
// one page table, consecutive page-table columns, equally spaced chunk bases,
// one layer stride, full descriptors but the last. Fills `out`, or returns
// false.
inline bool affine_form(const std::vector<XferDesc>& d, uint32_t page_tokens, PagedCopyPlan& out) {
    if (d.empty() || page_tokens == 0) return false;
    const XferDesc& a = d[0];
    const uint32_t pages = (a.n_tokens + page_tokens - 1) / page_tokens;
    if (pages == 0) return false;
    const uint64_t cs = d.size() > 1 ? d[1].chunk - a.chunk : 0;
    for (size_t i = 0; i < d.size(); ++i) {
        const XferDesc& x = d[i];
        const bool last = i + 1 == d.size();
        if (x.table != a.table || x.table_stride != a.table_stride || x.layer_stride != a.layer_stride) return false;
        if (x.first_page != a.first_page + uint32_t(i) * pages || x.chunk != a.chunk + i * cs) return false;
        if (last ? (x.n_tokens == 0 || x.n_tokens > pages * page_tokens) : x.n_tokens != pages * page_tokens)
            return false;
    }
    out.aff_pages = pages;
    out.aff_last_tokens = d.back().n_tokens;
    out.aff_first_page = a.first_page;
    out.aff_table_stride = a.table_stride;
    out.aff_table = a.table;
    out.aff_chunk0 = a.chunk;
    out.aff_chunk_stride = cs;
    out.aff_layer_stride = a.layer_stride;
    return true;
}

struct DevicePlan {
    size_t n_desc = 0;
    size_t variants = 0;
    uint32_t ppt_1 = 1, ppt_all = 1;
    uint32_t tiles_1 = 0, tiles_all = 0;
    uint64_t addr_or = 0;
    size_t off_tb1 = 0, off_tball = 0;
    DualPool* pool = nullptr;
    std::unique_ptr<DualBuffer> buf;
    std::vector<PagedCopyPlan> affine;  // per variant: aff_* fields (aff_pages 0: none)

    DevicePlan() = default;
    DevicePlan(const DevicePlan&) = delete;
    DevicePlan& operator=(const DevicePlan&) = delete;
    // The owner guarantees the device work reading the plan has finished.
    ~DevicePlan() {
        if (pool && buf) pool->release(std::move(buf));
    }

    void build(DualPool& p, const std::vector<std::vector<XferDesc>>& vars, uint32_t page_tokens,
               size_t page_bytes, uint32_t n_layers, cudaStream_t s) {
        variants = vars.size();
        n_desc = vars.empty() ? 0 : vars[0].size();
        if (n_desc == 0) return;
        ppt_1 = pages_per_tile_one_layer(page_bytes);
        ppt_all = pages_per_tile(page_bytes);
        auto tb1 = tile_prefix(vars[0], page_tokens, ppt_1, 1);
        auto tball = tile_prefix(vars[0], page_tokens, ppt_all, n_layers);
        tiles_1 = tb1.back();
        tiles_all = tball.back();
        const size_t desc_bytes = variants * n_desc * sizeof(XferDesc);
        off_tb1 = (desc_bytes + 15) & ~size_t(15);
        off_tball = off_tb1 + ((tb1.size() * 4 + 15) & ~size_t(15));
        const size_t total = off_tball + tball.size() * 4;
        if (pool && buf) pool->release(std::move(buf));
        pool = &p;
        buf = p.acquire(total);
        uint8_t* h = buf->host.host;
        addr_or = 0;
        for (size_t v = 0; v < variants; ++v) {
            std::memcpy(h + v * n_desc * sizeof(XferDesc), vars[v].data(), n_desc * sizeof(XferDesc));
            for (const auto& d : vars[v]) addr_or |= d.chunk | d.layer_stride;
        }
        affine.assign(variants, PagedCopyPlan{});
        for (size_t v = 0; v < variants; ++v) affine_form(vars[v], page_tokens, affine[v]);
        std::memcpy(h + off_tb1, tb1.data(), tb1.size() * 4);
        std::memcpy(h + off_tball, tball.data(), tball.size() * 4);
        // SM copy from the mapped pinned side: a copy-engine upload would queue
        // behind the layer transfers already in flight.
        TKV_CUDA(launch_sm_copy(buf->host.dev, buf->dev.ptr, total, s));
    }

    // Launch plan over [layer_begin, layer_begin + n_layers): the one-layer
    // tile prefix for n_layers == 1, the all-layer one otherwise (which must
    // then cover every layer of the build).
    PagedCopyPlan plan(size_t variant, uint32_t layer_begin, uint32_t n_layers) const {
        PagedCopyPlan p;
        p.descs = reinterpret_cast<const XferDesc*>(buf->dev.ptr) + variant * n_desc;
        const bool one = n_layers == 1;
        p.tile_base = reinterpret_cast<const uint32_t*>(buf->dev.ptr + (one ? off_tb1 : off_tball));
        p.n_desc = uint32_t(n_desc);
        p.total_tiles = one ? tiles_1 : tiles_all;
        p.layer_begin = layer_begin;
        p.n_layers = n_layers;
        p.pages_per_tile = one ? ppt_1 : ppt_all;
        p.addr_or = addr_or;
        if (one && ppt_1 == 1 && variant < affine.size() && affine[variant].aff_pages) {
            const PagedCopyPlan& f = affine[variant];
            p.aff_pages = f.aff_pages;
            p.aff_last_tokens = f.aff_last_tokens;
            p.aff_first_page = f.aff_first_page;
            p.aff_table_stride = f.aff_table_stride;
            p.aff_table = f.aff_table;
            p.aff_chunk0 = f.aff_chunk0;
            p.aff_chunk_stride = f.aff_chunk_stride;
            p.aff_layer_stride = f.aff_layer_stride;
        }
        return p;
    }
};

}  // namespace tkv
