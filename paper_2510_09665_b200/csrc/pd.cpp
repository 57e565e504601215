#include "pd.hpp"

#include <algorithm>
#include <map>
#include <memory>

#include "copy_plan.hpp"

namespace tkv {

// --- control plane: the contract of src/pd_staging.cpp:5-63 ---------------
// (register before push; an ordinal is filled once and a retransmit acks; no
// ordinal past the final one, and no final marker below a filled ordinal;
// await hands back the records in ordinal order and forgets the query;
// cancel wakes the awaiter with io_error)

Status PdStaging::register_query(QueryId id) {
    std::lock_guard lock(mu_);
    if (!landings_.emplace(id, std::make_shared<Landing>()).second)
        return Status{Errc::duplicate_key, "query " + std::to_string(id) + " is already registered"};
    return Status::success();
}

Status PdStaging::push(QueryId id, uint32_t ordinal, bool last, const PdRecord& rec) {
    std::lock_guard lock(mu_);
    const auto it = landings_.find(id);
    if (it == landings_.end()) return Status{Errc::unknown_query, "push for unregistered query " + std::to_string(id)};
    Landing& l = *it->second;
    if (l.final_known && ordinal > l.final_ordinal)
        return Status{Errc::protocol_error, "ordinal " + std::to_string(ordinal) + " past the final one"};
    if (last && !l.filled.empty() && l.highest > ordinal)
        return Status{Errc::protocol_error, "final ordinal " + std::to_string(ordinal) + " below a filled one"};
    if (last) {
        l.final_known = true;
        l.final_ordinal = ordinal;
    }
    if (l.filled.emplace(ordinal, rec).second) l.highest = l.filled.size() == 1 ? ordinal : std::max(l.highest, ordinal);
    if (l.done()) l.wake.notify_all();
    return Status::success();
}

Result<std::vector<PdRecord>> PdStaging::await(QueryId id) {
    std::unique_lock lock(mu_);
    const auto it = landings_.find(id);
    if (it == landings_.end()) return Status{Errc::unknown_query, "await for unregistered query " + std::to_string(id)};
    const std::shared_ptr<Landing> l = it->second;
    l->wake.wait(lock, [&] { return l->done() || l->cancelled; });
    const auto now = landings_.find(id);
    if (now != landings_.end() && now->second == l) landings_.erase(now);
    if (l->cancelled) return Status{Errc::io_error, "query " + std::to_string(id) + " was cancelled"};
    std::vector<PdRecord> out(l->filled.size());
    for (const auto& [ordinal, rec] : l->filled) out[ordinal] = rec;  // ordinals are exactly 0..final
    return out;
}

Status PdStaging::cancel(QueryId id) {
    std::lock_guard lock(mu_);
    const auto it = landings_.find(id);
    if (it == landings_.end()) return Status{Errc::unknown_query, "cancel for unregistered query " + std::to_string(id)};
    it->second->cancelled = true;
    it->second->wake.notify_all();
    return Status::success();
}

size_t PdStaging::registered() const {
    std::lock_guard lock(mu_);
    return landings_.size();
}

// --- data plane ------------------------------------------------------------

namespace {
// Plan buffers and the copy-engine stream are per device: a process may drive
// several GPUs (one engine per device), and a pooled buffer or a stream
// belongs to the device that was current when it was created.
DualPool& pd_plan_pool() {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<DualPool>> pools;
    int dev = 0;
    TKV_CUDA(cudaGetDevice(&dev));
    std::lock_guard lock(mu);
    auto& p = pools[dev];
    if (!p) p = std::make_unique<DualPool>();
    return *p;
}
cudaStream_t pd_ce_stream() {
    thread_local std::map<int, Stream> streams;
    int dev = 0;
    TKV_CUDA(cudaGetDevice(&dev));
    auto it = streams.find(dev);
    if (it == streams.end()) it = streams.emplace(dev, Stream::create()).first;
    return it->second;
}
}  // namespace

namespace {
// Records (where each chunk lands) and K1 descriptors writing chunk i at
// base + i * chunk_stride, after the reference's readability checks.
Status pd_describe(PagedKVStore& pages, QueryId query, size_t n_tokens, size_t chunk_size,
                   uint64_t landing, uint64_t base, uint64_t chunk_stride, cudaStream_t stream,
                   std::vector<PdRecord>& recs, std::vector<XferDesc>& descs, bool check_layers = true) {
    TKV_CUDA(cudaSetDevice(pages.device()));
    const auto& spec = pages.spec();
    const uint32_t pt = spec.page_tokens;
    const size_t bpt = spec.bytes_per_token_per_layer;
    if (chunk_size == 0 || chunk_size % pt) return Status{Errc::invalid_argument, "chunk size"};
    auto t = pages.device_table(query, stream);
    if (!t.ok()) return t.status();
    // Per chunk, its layers' readability then its landing size (the first
    // failure in that order is the result). Chunk 0 is the largest, so a
    // size failure is chunk 0's, after chunk 0's readability.
    std::vector<PagedKVStore::PageSpan> spans;
    for (size_t start = 0; start < n_tokens; start += chunk_size)
        spans.push_back({start / pt, std::min(chunk_size, n_tokens - start)});
    const bool too_big = !spans.empty() && uint64_t(spec.num_layers) * spans[0].token_count * bpt > chunk_stride;
    if (check_layers) {
        if (too_big) spans.resize(1);
        Status st = pages.check_readable_spans(query, spans, 0, spec.num_layers);
        if (!st.ok()) return st;
    }
    if (too_big) return Status{Errc::size_mismatch, "landing slot too small"};
    for (size_t start = 0, i = 0; start < n_tokens; start += chunk_size, ++i) {
        const size_t n = std::min(chunk_size, n_tokens - start);
        const uint64_t bytes = uint64_t(spec.num_layers) * n * bpt;
        recs.push_back(PdRecord{landing + i * chunk_stride, bytes, uint32_t(n), uint32_t(start)});
        XferDesc x;
        x.chunk = base + i * chunk_stride;
        x.layer_stride = uint64_t(n) * bpt;
        x.table = t.value().ptr;
        x.table_stride = t.value().stride;
        x.first_page = uint32_t(start / pt);
        x.n_tokens = uint32_t(n);
        descs.push_back(x);
    }
    return Status::success();
}
}  // namespace

Result<std::vector<PdRecord>> pd_send_chunks(PagedKVStore& pages, QueryId query, size_t n_tokens,
                                             size_t chunk_size, uint64_t landing,
                                             uint64_t chunk_stride, cudaStream_t stream, int ctas) {
    const auto& spec = pages.spec();
    std::vector<PdRecord> recs;
    std::vector<XferDesc> descs;
    Status st = pd_describe(pages, query, n_tokens, chunk_size, landing, landing, chunk_stride, stream, recs, descs);
    if (!st.ok()) return st;
    if (descs.empty()) return recs;
    const uint32_t pt = spec.page_tokens;
    DevicePlan plan;
    plan.build(pd_plan_pool(), {descs}, pt, pages.page_bytes(), spec.num_layers, stream);
    TKV_CUDA(launch_paged_copy(pages.layout(), plan.plan(0, 0, spec.num_layers), CopyDir::gather,
                               ctas, stream));
    TKV_CUDA(cudaStreamSynchronize(stream));  // bytes landed before any ordinal is pushed
    return recs;
}

Result<std::vector<PdRecord>> pd_send_chunks_staged(PagedKVStore& pages, QueryId query, size_t n_tokens,
                                                    size_t chunk_size, uint64_t landing,
                                                    uint64_t chunk_stride, uint64_t staging,
                                                    cudaStream_t stream, uint64_t group_bytes) {
    const auto& spec = pages.spec();
    std::vector<PdRecord> recs;
    std::vector<XferDesc> descs;
    Status st = pd_describe(pages, query, n_tokens, chunk_size, landing, staging, chunk_stride, stream, recs, descs);
    if (!st.ok()) return st;
    if (descs.empty()) return recs;
    const uint32_t pt = spec.page_tokens;
    const size_t per_group = std::max<size_t>(1, group_bytes / chunk_stride);
    std::vector<std::vector<XferDesc>> groups;
    for (size_t i = 0; i < descs.size(); i += per_group)
        groups.emplace_back(descs.begin() + i, descs.begin() + std::min(descs.size(), i + per_group));
    std::vector<DevicePlan> plans(groups.size());  // group sizes differ: one plan each
    cudaStream_t ce = pd_ce_stream();
    std::vector<Event> done(groups.size());
    for (size_t g = 0; g < groups.size(); ++g) {
        plans[g].build(pd_plan_pool(), {groups[g]}, pt, pages.page_bytes(), spec.num_layers, stream);
        TKV_CUDA(launch_paged_copy(pages.layout(), plans[g].plan(0, 0, spec.num_layers),
                                   CopyDir::gather, 0, stream));
        done[g].record(stream);
        done[g].wait_on(ce);
        const size_t first = g * per_group, last = first + groups[g].size() - 1;
        const uint64_t bytes = (last - first) * chunk_stride + recs[last].bytes;
        TKV_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(landing + first * chunk_stride),
                                 reinterpret_cast<const void*>(staging + first * chunk_stride), bytes,
                                 cudaMemcpyDefault, ce));
    }
    TKV_CUDA(cudaStreamSynchronize(ce));  // bytes landed before any ordinal is pushed
    TKV_CUDA(cudaStreamSynchronize(stream));
    return recs;
}

PdLayerSender::PdLayerSender(PagedKVStore& pages, QueryId query, size_t n_tokens, size_t unit_tokens,
                             uint64_t landing, uint64_t unit_stride)
    : pages_(pages), query_(query), n_tokens_(n_tokens), unit_tokens_(unit_tokens) {
    TKV_CUDA(cudaSetDevice(pages.device()));
    stream_ = Stream::create();
    const auto& spec = pages.spec();
    sent_.assign(spec.num_layers, false);
    std::vector<XferDesc> descs;
    status_ = pd_describe(pages, query, n_tokens, unit_tokens, landing, landing, unit_stride, stream_, recs_, descs,
                          /*check_layers=*/false);
    if (!status_.ok() || descs.empty()) return;
    plan_ = std::make_unique<DevicePlan>();
    plan_->build(pd_plan_pool(), {descs}, spec.page_tokens, pages.page_bytes(), spec.num_layers, stream_);
}

PdLayerSender::~PdLayerSender() {
    try {
        TKV_CUDA(cudaStreamSynchronize(stream_));  // the plan is read by launches in flight
    } catch (...) {
    }
}

Status PdLayerSender::send_layer(uint32_t layer, cudaStream_t engine_stream) {
    if (!status_.ok()) return status_;
    const auto& spec = pages_.spec();
    if (layer >= spec.num_layers) return Status{Errc::invalid_argument, "layer out of range"};
    if (sent_[layer]) return Status{Errc::duplicate_key, "layer already sent"};
    const uint32_t pt = spec.page_tokens;
    {  // the engine computed this layer (check_readable)
        std::vector<PagedKVStore::PageSpan> spans;
        spans.reserve(recs_.size());
        for (const auto& r : recs_) spans.push_back({r.first_token / pt, r.token_count});
        Status st = pages_.check_readable_spans(query_, spans, layer, layer + 1);
        if (!st.ok()) return st;
    }
    sent_[layer] = true;
    if (!plan_) return Status::success();
    TKV_CUDA(cudaSetDevice(pages_.device()));
    Event computed;
    computed.record(engine_stream);
    computed.wait_on(stream_);
    TKV_CUDA(launch_paged_copy(pages_.layout(), plan_->plan(0, layer, 1), CopyDir::gather, 0, stream_));
    return Status::success();
}

Result<std::vector<PdRecord>> PdLayerSender::finish() {
    if (!status_.ok()) return status_;
    for (bool s : sent_)
        if (!s) return Status{Errc::invalid_argument, "a layer was not sent"};
    TKV_CUDA(cudaStreamSynchronize(stream_));  // every layer landed before any ordinal is pushed
    return recs_;
}

Status pd_land_chunks(PagedKVStore& pages, QueryId query, const std::vector<PdRecord>& records,
                      cudaStream_t stream, int ctas) {
    TKV_CUDA(cudaSetDevice(pages.device()));
    const auto& spec = pages.spec();
    const uint32_t pt = spec.page_tokens;
    const size_t bpt = spec.bytes_per_token_per_layer;
    auto t = pages.device_table(query, stream);
    if (!t.ok()) return t.status();
    // Per record: alignment, size, then every layer's pages writable; the
    // first failure in that order is the result (the page checks of the
    // records before the first malformed one run in one batch).
    size_t bad = records.size();
    Status bad_st;
    for (size_t i = 0; i < records.size() && bad == records.size(); ++i) {
        const auto& r = records[i];
        if (r.first_token % pt)
            bad = i, bad_st = Status{Errc::invalid_argument, "record not page aligned"};
        else if (r.bytes != uint64_t(spec.num_layers) * r.token_count * bpt)
            bad = i, bad_st = Status{Errc::size_mismatch, "pushed record size"};  // sim_engine.cpp:461-462
    }
    std::vector<PagedKVStore::PageSpan> spans;
    spans.reserve(bad);
    for (size_t i = 0; i < bad; ++i) spans.push_back({records[i].first_token / pt, records[i].token_count});
    if (Status st = pages.check_writable_spans(query, spans, 0, spec.num_layers); !st.ok()) return st;
    if (bad < records.size()) return bad_st;
    std::vector<XferDesc> descs;
    for (const auto& r : records) {
        XferDesc x;
        x.chunk = r.addr;
        x.layer_stride = uint64_t(r.token_count) * bpt;
        x.table = t.value().ptr;
        x.table_stride = t.value().stride;
        x.first_page = r.first_token / pt;
        x.n_tokens = r.token_count;
        descs.push_back(x);
    }
    if (descs.empty()) return Status::success();
    DevicePlan plan;
    plan.build(pd_plan_pool(), {descs}, pt, pages.page_bytes(), spec.num_layers, stream);
    TKV_CUDA(launch_paged_copy(pages.layout(), plan.plan(0, 0, spec.num_layers),
                               CopyDir::scatter, ctas, stream));
    pages.mark_spans_populated(query, spans, 0, spec.num_layers);
    TKV_CUDA(cudaStreamSynchronize(stream));  // plan buffers are freed on return
    return Status::success();
}

Status enable_peer_access(int device, int peer) {
    if (device == peer) return Status::success();
    int can = 0;
    TKV_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
    if (!can) return Status{Errc::invalid_argument, "no peer access between devices"};
    int prev = 0;
    TKV_CUDA(cudaGetDevice(&prev));
    TKV_CUDA(cudaSetDevice(device));
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    cudaSetDevice(prev);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return Status::success();
    }
    TKV_CUDA(e);
    return Status::success();
}

}  // namespace tkv
