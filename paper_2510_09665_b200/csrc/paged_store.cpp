#include "paged_store.hpp"

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>

namespace tkv {

PagedKVStore::PagedKVStore(ModelSpec spec, uint32_t num_pages, int device)
    : spec_(std::move(spec)), device_(device) {
    if (device_ < 0) TKV_CUDA(cudaGetDevice(&device_));
    TKV_CUDA(cudaSetDevice(device_));
    pool_.reserve(std::max<size_t>(1, size_t(num_pages) * spec_.page_bytes()));
    page_word_.assign(num_pages, layer_word(kNoLayer));
    // the top of the stack is the last element: descending ids put page 0 there
    free_ids_.resize(num_pages);
    std::iota(free_ids_.rbegin(), free_ids_.rend(), PageId(0));
    free_top_ = num_pages;
    io_stream_ = Stream::create();
}

Result<std::vector<PageId>> PagedKVStore::alloc_pages(QueryId query, size_t n) {
    std::lock_guard lock(mu_);
    if (n > free_top_)
        return Status{Errc::out_of_pages,
                      "alloc_pages: " + std::to_string(n) + " requested, " + std::to_string(free_top_) + " available"};
    // the n topmost ids, topmost first (the order a pop loop would give)
    std::vector<PageId> got(free_ids_.rbegin() + std::ptrdiff_t(free_ids_.size() - free_top_),
                            free_ids_.rbegin() + std::ptrdiff_t(free_ids_.size() - free_top_ + n));
    free_top_ -= n;
    for (PageId id : got) page_word_[id] = kAllocated | layer_word(kNoLayer);
    QueryPages& q = queries_[query];
    q.allocated = true;
    q.owned.insert(q.owned.end(), got.begin(), got.end());
    return got;
}

void PagedKVStore::bind_layer(QueryId query, uint32_t layer, const std::vector<PageId>& pages) {
    std::lock_guard lock(mu_);
    QueryPages& q = queries_[query];
    if (q.layers.size() <= layer) q.layers.resize(size_t(layer) + 1);
    q.layers[layer] = pages;
    q.dirty = true;
    for (PageId id : pages) page_word_[id] = (page_word_[id] & ~0xffffffffull) | layer_word(layer);
}

Status PagedKVStore::admit(QueryId query, size_t tokens) {
    const size_t blocks = (tokens + spec_.page_tokens - 1) / spec_.page_tokens;
    auto got = alloc_pages(query, blocks * spec_.num_layers);
    if (!got.ok()) return got.status();
    const std::vector<PageId>& ids = got.value();
    for (uint32_t l = 0; l < spec_.num_layers; ++l)
        bind_layer(query, l, std::vector<PageId>(ids.begin() + std::ptrdiff_t(size_t(l) * blocks),
                                                 ids.begin() + std::ptrdiff_t(size_t(l + 1) * blocks)));
    return Status::success();
}

std::vector<PageId> PagedKVStore::layer_pages(QueryId query, uint32_t layer) const {
    std::lock_guard lock(mu_);
    const auto it = queries_.find(query);
    return it != queries_.end() && layer < it->second.layers.size() ? it->second.layers[layer]
                                                                    : std::vector<PageId>{};
}

std::vector<PageId> PagedKVStore::release_query(QueryId query) {
    std::lock_guard lock(mu_);
    auto it = queries_.find(query);
    if (it == queries_.end() || !it->second.allocated) return {};  // page lists without pages stay
    QueryPages q = std::move(it->second);
    queries_.erase(it);
    // the engine releases a query after its transfers finished: its table
    // mirrors go back to the pool
    if (q.buf) table_pool_.release(std::move(q.buf));
    for (auto& r : q.retired) table_pool_.release(std::move(r));
    for (PageId id : q.owned) {
        page_word_[id] = layer_word(kNoLayer);
        free_ids_[free_top_++] = id;
    }
    return std::move(q.owned);
}

size_t PagedKVStore::free_page_count() const {
    std::lock_guard lock(mu_);
    return free_top_;
}

size_t PagedKVStore::allocated_page_count() const {
    std::lock_guard lock(mu_);
    return page_word_.size() - free_top_;
}

void PagedKVStore::mark_populated(PageId id, uint32_t layer) {
    std::lock_guard lock(mu_);
    page_word_[id] = (page_word_[id] & kAllocated) | kPopulated | layer_word(layer);
}

bool PagedKVStore::populated(PageId id) const {
    std::lock_guard lock(mu_);
    return (page_word_[id] & kPopulated) != 0;
}

PagedLayout PagedKVStore::layout() const {
    PagedLayout L;
    L.base = reinterpret_cast<uint64_t>(pool_.ptr);
    L.page_stride = page_bytes();
    L.token_stride = spec_.bytes_per_token_per_layer;
    L.plane_bytes = spec_.bytes_per_token_per_layer;
    L.plane_stride = 0;
    L.n_planes = 1;
    L.page_tokens = spec_.page_tokens;
    L.bpt = spec_.bytes_per_token_per_layer;
    L.shared_table = 0;
    return L;
}

Result<PagedKVStore::DeviceTable> PagedKVStore::device_table(QueryId query, cudaStream_t stream) {
    std::lock_guard lock(mu_);
    auto it = queries_.find(query);
    if (it == queries_.end()) return Status{Errc::unknown_query, "query has no page table"};
    QueryPages& t = it->second;
    if (t.dirty) {
        size_t stride = 1;
        for (const auto& l : t.layers) stride = std::max(stride, l.size());
        const size_t rows = std::max<size_t>(spec_.num_layers, t.layers.size());
        const size_t bytes = rows * stride * sizeof(int32_t);
        // A re-bound table gets a fresh block: the old one may still feed an
        // in-flight upload or kernel, so it is only recycled at release.
        auto fresh = table_pool_.acquire(bytes);
        if (t.buf) t.retired.push_back(std::move(t.buf));
        t.buf = std::move(fresh);
        auto* h = reinterpret_cast<int32_t*>(t.buf->host.host);
        std::fill(h, h + rows * stride, -1);
        for (size_t l = 0; l < t.layers.size(); ++l)
            std::copy(t.layers[l].begin(), t.layers[l].end(), h + l * stride);
        // SM copy from the mapped pinned side (not behind in-flight CE transfers)
        TKV_CUDA(launch_sm_copy(t.buf->host.dev, t.buf->dev.ptr, bytes, stream));
        t.stride = uint32_t(stride);
        t.dirty = false;
    }
    return DeviceTable{reinterpret_cast<const int32_t*>(t.buf->dev.ptr), t.stride};
}

namespace {
std::string page_msg(PageId id, uint32_t layer) {
    return "page " + std::to_string(id) + " holds no data of layer " + std::to_string(layer);
}
}  // namespace

// paged_store.cpp:94-111: capacity, then every page in order (range, then
// populated with this layer's data)
Status PagedKVStore::check_readable(const std::vector<PageId>& pages, uint32_t layer,
                                    size_t token_count) const {
    if (token_count > pages.size() * spec_.page_tokens)
        return Status{Errc::size_mismatch, std::to_string(token_count) + " tokens do not fit " +
                                               std::to_string(pages.size()) + " pages"};
    std::lock_guard lock(mu_);
    for (PageId id : pages) {
        if (id >= page_word_.size()) return Status{Errc::invalid_argument, "page " + std::to_string(id) + " not in the pool"};
        if (!page_holds(id, layer)) return Status{Errc::unpopulated_page, page_msg(id, layer)};
    }
    return Status::success();
}

const std::vector<PageId>* PagedKVStore::span_list(QueryId query, uint32_t layer, size_t first_page,
                                                   size_t token_count, size_t& end) const {
    const auto it = queries_.find(query);
    if (it == queries_.end() || it->second.layers.size() <= layer) return nullptr;
    const auto& list = it->second.layers[layer];
    end = first_page + (token_count + spec_.page_tokens - 1) / spec_.page_tokens;
    return end <= list.size() ? &list : nullptr;
}

Status PagedKVStore::check_readable_span(QueryId query, uint32_t layer, size_t first_page,
                                         size_t token_count) const {
    std::lock_guard lock(mu_);
    return readable_locked(query, layer, first_page, token_count);
}

Status PagedKVStore::readable_locked(QueryId query, uint32_t layer, size_t first_page,
                                     size_t token_count) const {
    size_t end = 0;
    const auto* list = span_list(query, layer, first_page, token_count, end);
    if (list == nullptr)
        return Status{Errc::size_mismatch, "layer " + std::to_string(layer) + " has no pages for " +
                                               std::to_string(token_count) + " tokens"};
    for (size_t i = first_page; i < end; ++i)
        if (!page_holds((*list)[i], layer)) return Status{Errc::unpopulated_page, page_msg((*list)[i], layer)};
    return Status::success();
}

Status PagedKVStore::check_writable_span(QueryId query, uint32_t layer, size_t first_page,
                                         size_t token_count) const {
    std::lock_guard lock(mu_);
    return writable_locked(query, layer, first_page, token_count);
}

Status PagedKVStore::writable_locked(QueryId query, uint32_t layer, size_t first_page,
                                     size_t token_count) const {
    size_t end = 0;
    const auto* list = span_list(query, layer, first_page, token_count, end);
    if (list == nullptr) return Status{Errc::size_mismatch, "span larger than the bound pages"};
    for (size_t i = first_page; i < end; ++i) {
        const PageId id = (*list)[i];
        if (id >= page_word_.size()) return Status{Errc::invalid_argument, "page " + std::to_string(id) + " not in the pool"};
        if (!(page_word_[id] & kAllocated))
            return Status{Errc::invalid_argument, "page " + std::to_string(id) + " is not allocated"};
    }
    return Status::success();
}

void PagedKVStore::mark_span_populated(QueryId query, uint32_t layer, size_t first_page,
                                       size_t token_count) {
    std::lock_guard lock(mu_);
    populate_locked(query, layer, first_page, token_count);
}

Status PagedKVStore::check_readable_spans(QueryId query, const std::vector<PageSpan>& spans, uint32_t l0,
                                          uint32_t l1) const {
    std::lock_guard lock(mu_);
    for (const auto& sp : spans)
        for (uint32_t l = l0; l < l1; ++l) {
            Status st = readable_locked(query, l, sp.first_page, sp.token_count);
            if (!st.ok()) return st;
        }
    return Status::success();
}

Status PagedKVStore::check_writable_spans(QueryId query, const std::vector<PageSpan>& spans, uint32_t l0,
                                          uint32_t l1) const {
    std::lock_guard lock(mu_);
    for (const auto& sp : spans)
        for (uint32_t l = l0; l < l1; ++l) {
            Status st = writable_locked(query, l, sp.first_page, sp.token_count);
            if (!st.ok()) return st;
        }
    return Status::success();
}

void PagedKVStore::mark_spans_populated(QueryId query, const std::vector<PageSpan>& spans, uint32_t l0,
                                        uint32_t l1) {
    std::lock_guard lock(mu_);
    for (const auto& sp : spans)
        for (uint32_t l = l0; l < l1; ++l) populate_locked(query, l, sp.first_page, sp.token_count);
}

void PagedKVStore::populate_locked(QueryId query, uint32_t layer, size_t first_page, size_t token_count) {
    const auto it = queries_.find(query);
    if (it == queries_.end() || it->second.layers.size() <= layer) return;
    const auto& list = it->second.layers[layer];
    const size_t end = std::min(list.size(), first_page + (token_count + spec_.page_tokens - 1) / spec_.page_tokens);
    for (size_t i = first_page; i < end; ++i)
        page_word_[list[i]] = (page_word_[list[i]] & kAllocated) | kPopulated | layer_word(layer);
}

Status PagedKVStore::copy_through_pages(const std::vector<PageId>& pages, uint32_t layer,
                               size_t token_count, uint8_t* host, CopyDir dir) {
    if (token_count == 0) return Status::success();
    std::lock_guard lock(io_mu_);
    TKV_CUDA(cudaSetDevice(device_));
    const size_t bpt = spec_.bytes_per_token_per_layer;
    const size_t bytes = token_count * bpt;
    const size_t used_pages = (token_count + spec_.page_tokens - 1) / spec_.page_tokens;
    // Device scratch: [XferDesc][tile_base x2][table]
    const size_t table_off = 64;
    const size_t scratch = table_off + used_pages * sizeof(int32_t);
    io_dev_.reserve(scratch);
    io_host_.reserve(scratch + bytes + 16);
    uint8_t* payload = io_host_.host + ((scratch + 15) & ~size_t(15));
    uint8_t* payload_dev = io_host_.dev + ((scratch + 15) & ~size_t(15));

    const uint32_t ppt = std::max<uint32_t>(1, std::min<uint32_t>(64, 65536 / page_bytes()));
    XferDesc d;
    d.chunk = reinterpret_cast<uint64_t>(payload_dev);
    d.layer_stride = 0;
    d.table = reinterpret_cast<const int32_t*>(io_dev_.ptr + table_off);
    d.table_stride = uint32_t(used_pages);
    d.first_page = 0;
    d.n_tokens = uint32_t(token_count);
    uint32_t tiles = tiles_for(d.n_tokens, spec_.page_tokens, ppt, 1);
    std::memcpy(io_host_.host, &d, sizeof d);
    uint32_t tb[2] = {0, tiles};
    std::memcpy(io_host_.host + 40, tb, sizeof tb);
    auto* tab = reinterpret_cast<int32_t*>(io_host_.host + table_off);
    for (size_t i = 0; i < used_pages; ++i) tab[i] = int32_t(pages[i]);
    if (dir == CopyDir::scatter) std::memcpy(payload, host, bytes);
    TKV_CUDA(cudaMemcpyAsync(io_dev_.ptr, io_host_.host, scratch, cudaMemcpyHostToDevice,
                             io_stream_));
    PagedLayout L = layout();
    L.shared_table = 1;  // the single table row serves the requested layer
    PagedCopyPlan P;
    P.descs = reinterpret_cast<const XferDesc*>(io_dev_.ptr);
    P.tile_base = reinterpret_cast<const uint32_t*>(io_dev_.ptr + 40);
    P.n_desc = 1;
    P.total_tiles = tiles;
    P.layer_begin = layer;
    P.n_layers = 1;
    P.pages_per_tile = ppt;
    P.addr_or = d.chunk;
    TKV_CUDA(launch_paged_copy(L, P, dir, 0, io_stream_));
    TKV_CUDA(cudaStreamSynchronize(io_stream_));
    if (dir == CopyDir::gather) std::memcpy(host, payload, bytes);
    return Status::success();
}

Status PagedKVStore::gather_tokens_into(const std::vector<PageId>& pages, uint32_t layer,
                                        size_t token_count, uint8_t* out, size_t out_bytes) {
    if (out_bytes != token_count * spec_.bytes_per_token_per_layer)
        return Status{Errc::size_mismatch, "gather output size"};
    Status st = check_readable(pages, layer, token_count);
    if (!st.ok()) return st;
    return copy_through_pages(pages, layer, token_count, out, CopyDir::gather);
}

Result<std::vector<uint8_t>> PagedKVStore::gather_tokens(const std::vector<PageId>& pages,
                                                         uint32_t layer, size_t token_count) {
    std::vector<uint8_t> out(token_count * spec_.bytes_per_token_per_layer);
    Status st = gather_tokens_into(pages, layer, token_count, out.data(), out.size());
    if (!st.ok()) return st;
    return out;
}

Status PagedKVStore::scatter_tokens(const uint8_t* buf, size_t buf_bytes,
                                    const std::vector<PageId>& pages, uint32_t layer,
                                    size_t token_count) {
    if (buf_bytes != token_count * spec_.bytes_per_token_per_layer)
        return Status{Errc::size_mismatch, "scatter input size"};
    if (token_count > pages.size() * spec_.page_tokens)
        return Status{Errc::size_mismatch, "span larger than the bound pages"};
    {
        std::lock_guard lock(mu_);
        for (PageId id : pages) {
            if (id >= page_word_.size())
                return Status{Errc::invalid_argument, "page " + std::to_string(id) + " not in the pool"};
            if (!(page_word_[id] & kAllocated))
                return Status{Errc::invalid_argument, "page " + std::to_string(id) + " is not allocated"};
        }
    }
    Status st = copy_through_pages(pages, layer, token_count, const_cast<uint8_t*>(buf), CopyDir::scatter);
    if (!st.ok()) return st;
    const size_t used = (token_count + spec_.page_tokens - 1) / spec_.page_tokens;
    for (size_t i = 0; i < used; ++i) mark_populated(pages[i], layer);
    return Status::success();
}

}  // namespace tkv
