// Engine-resident paged KV memory on the device (mirror of
// include/tierkv/paged_store.hpp:19-82).
//
// The reference's observable contract — which page ids an allocation returns
// (last freed first; page 0 first in a fresh pool, paged_store.cpp:8-14),
// per-(query, layer) page lists, and the error codes of its checks — with a
// B200 layout: the pool is ONE cudaMalloc slab in HBM (page p at base +
// p * page_bytes), each query's page lists are mirrored into a device page
// table [num_layers][blocks] of int32 that the K1/K2/K4 kernels index
// directly, and the host side keeps one packed word per page plus one
// record per query.
#pragma once

#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"

namespace tkv {

class PagedKVStore {
public:
    PagedKVStore(ModelSpec spec, uint32_t num_pages, int device = -1);

    const ModelSpec& spec() const { return spec_; }
    size_t page_bytes() const { return spec_.page_bytes(); }
    uint32_t pool_pages() const { return uint32_t(page_word_.size()); }
    int device() const { return device_; }

    Result<std::vector<PageId>> alloc_pages(QueryId query, size_t n);
    void bind_layer(QueryId query, uint32_t layer, const std::vector<PageId>& pages);
    // SimEngine::admit (src/sim_engine.cpp:83-95): blocks*L pages for a
    // `tokens`-long sequence, layer l bound to pages [l*blocks, (l+1)*blocks).
    Status admit(QueryId query, size_t tokens);
    std::vector<PageId> layer_pages(QueryId query, uint32_t layer) const;
    std::vector<PageId> release_query(QueryId query);
    size_t free_page_count() const;
    size_t allocated_page_count() const;

    uint8_t* page_data(PageId id) const { return pool_.ptr + size_t(id) * page_bytes(); }
    void mark_populated(PageId id, uint32_t layer);
    bool populated(PageId id) const;

    // --- device view -------------------------------------------------------
    PagedLayout layout() const;
    struct DeviceTable {
        const int32_t* ptr = nullptr;
        uint32_t stride = 0;  // entries per layer row
    };
    // Uploads the query's page lists if they changed since the last upload
    // (stream-ordered on `stream`). Fails for an unknown query.
    Result<DeviceTable> device_table(QueryId query, cudaStream_t stream);

    // --- checks shared by every data path (paged_store.cpp:94-111,147-162) --
    // Pages [first, first+ceil(n/pt)) of (query, layer) exist, are owned and
    // hold `layer` data (gather side).
    Status check_readable_span(QueryId query, uint32_t layer, size_t first_page,
                               size_t token_count) const;
    // Same pages exist and are owned (scatter side).
    Status check_writable_span(QueryId query, uint32_t layer, size_t first_page,
                               size_t token_count) const;
    // Marks the pages covering [first_page, +ceil(n/pt)) of the span populated.
    void mark_span_populated(QueryId query, uint32_t layer, size_t first_page, size_t token_count);
    // The three above over many spans of one query and layers [l0, l1),
    // span by span and layer by layer within a span (the order, hence the
    // first error, of one call per (span, layer)), under one lock: a PD
    // send / land of a 32K-token prompt is 128 chunks x 80 layers.
    struct PageSpan {
        size_t first_page = 0, token_count = 0;
    };
    Status check_readable_spans(QueryId query, const std::vector<PageSpan>& spans, uint32_t l0, uint32_t l1) const;
    Status check_writable_spans(QueryId query, const std::vector<PageSpan>& spans, uint32_t l0, uint32_t l1) const;
    void mark_spans_populated(QueryId query, const std::vector<PageSpan>& spans, uint32_t l0, uint32_t l1);

    // --- reference-shaped single-layer host API (tests, tools) -------------
    // Synchronous: these move bytes between host memory and pages with the
    // K1/K2 kernels on an internal stream.
    Status gather_tokens_into(const std::vector<PageId>& pages, uint32_t layer,
                              size_t token_count, uint8_t* out, size_t out_bytes);
    Result<std::vector<uint8_t>> gather_tokens(const std::vector<PageId>& pages, uint32_t layer,
                                               size_t token_count);
    Status scatter_tokens(const uint8_t* buf, size_t buf_bytes, const std::vector<PageId>& pages,
                          uint32_t layer, size_t token_count);

private:
    // One 64-bit word per page: the layer it holds (low 32 bits) and two
    // flags. The owning query is known from its QueryPages record; a page
    // only needs "allocated" for the scatter-side check.
    static constexpr uint64_t kAllocated = 1ull << 32;
    static constexpr uint64_t kPopulated = 1ull << 33;
    static constexpr uint32_t kNoLayer = ~uint32_t(0);
    static uint64_t layer_word(uint32_t layer) { return uint64_t(layer); }
    bool page_holds(PageId id, uint32_t layer) const {  // caller holds mu_
        const uint64_t w = page_word_[id];
        return (w & kPopulated) && uint32_t(w) == layer;
    }
    // Everything the store knows about one query: the pages it allocated (in
    // allocation order), its per-layer page lists and their device mirror.
    struct QueryPages {
        bool allocated = false;  // alloc_pages ran for it (possibly with n = 0)
        std::vector<PageId> owned;
        std::vector<std::vector<PageId>> layers;
        bool dirty = true;
        uint32_t stride = 0;
        std::unique_ptr<DualBuffer> buf;  // pooled pinned mirror + device table
        std::vector<std::unique_ptr<DualBuffer>> retired;  // earlier uploads, freed at release
    };
    // span [first, first + ceil(n / page_tokens)) of (query, layer), or null
    const std::vector<PageId>* span_list(QueryId query, uint32_t layer, size_t first_page, size_t token_count,
                                         size_t& end) const;
    // bodies of the span checks / mark; caller holds mu_
    Status readable_locked(QueryId query, uint32_t layer, size_t first_page, size_t token_count) const;
    Status writable_locked(QueryId query, uint32_t layer, size_t first_page, size_t token_count) const;
    void populate_locked(QueryId query, uint32_t layer, size_t first_page, size_t token_count);

    Status check_readable(const std::vector<PageId>& pages, uint32_t layer,
                          size_t token_count) const;
    Status copy_through_pages(const std::vector<PageId>& pages, uint32_t layer, size_t token_count,
                              uint8_t* host, CopyDir dir);

    ModelSpec spec_;
    int device_;
    DeviceBuffer pool_;
    std::vector<uint64_t> page_word_;
    // LIFO of free page ids: free_ids_[0, free_top_) with the next page to
    // hand out at the top (page 0 first after construction)
    std::vector<PageId> free_ids_;
    size_t free_top_ = 0;
    DualPool table_pool_;  // declared before queries_: outlives their mirrors
    std::unordered_map<QueryId, QueryPages> queries_;
    mutable std::mutex mu_;

    std::mutex io_mu_;  // serialises the synchronous host API
    Stream io_stream_;
    PinnedBuffer io_host_;
    DeviceBuffer io_dev_;
};

}  // namespace tkv
