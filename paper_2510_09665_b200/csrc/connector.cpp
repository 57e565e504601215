#include "connector.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "copy_plan.hpp"
#include "host_copy.hpp"

namespace tkv {

namespace {

// Per-layer events are timing-capable so a batch can report its device
// timeline (tkv_meta_timeline) without a profiler.
void make_events(std::vector<Event>& v, size_t n) {
    v.clear();
    v.reserve(n);
    for (size_t i = 0; i < n; ++i) v.emplace_back(true);
}

float elapsed(const Event& a, const Event& b) {
    float ms = -1.f;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
        cudaGetLastError();
        return -1.f;
    }
    return ms;
}

// Set once a batch's load shares are released (after its last scatter).
struct ReleaseState {
    std::mutex m;
    std::condition_variable cv;
    bool done = false;
    void wait() {
        std::unique_lock lock(m);
        cv.wait(lock, [&] { return done; });
    }
};
struct ReleaseCtx {
    TieredStore* store;
    std::vector<Digest> digests;
    std::shared_ptr<ReleaseState> state;
};
void CUDART_CB release_cb(void* p) {
    auto* c = static_cast<ReleaseCtx*>(p);
    for (const auto& d : c->digests) c->store->release(d);
    if (c->state) {
        {
            std::lock_guard lock(c->state->m);
            c->state->done = true;
        }
        c->state->cv.notify_all();
    }
    delete c;
}

struct CommitCtx {
    TieredStore* store;
    std::vector<Digest> digests;
    std::atomic<bool>* committed;
    std::vector<Digest> touches;  // the reference's LRU touch order for the batch
    std::shared_ptr<void> keep;   // device-read buffers (a launch plan) freed after the copy
};
void CUDART_CB commit_cb(void* p) {
    auto* c = static_cast<CommitCtx*>(p);
    c->store->commit_batch(c->digests, c->touches);
    if (c->committed) c->committed->store(true);
    delete c;
}

}  // namespace

namespace detail {

struct PerQueryState {
    size_t loaded = 0;
    std::vector<std::pair<ChunkKey, Status>> store_results;
};

struct LoadItem {
    QueryId id;
    Digest digest;
    SlotRead slot;
    ChunkSpan span;
    uint32_t record_tokens;
    size_t staging_off;
};

struct StoreItem {
    size_t plan;
    size_t desc;
    Status status;  // reservation outcome
    SlotWrite w;
    size_t staging_off = 0;  // copy-engine path: offset in one staging layer
    size_t rows = 0;         // span length
    size_t record_tokens = 0;
};

struct BatchState {
    Connector* conn = nullptr;
    TransferMode mode = TransferMode::layerwise;
    uint32_t num_layers = 0;
    std::vector<QueryPlan> plans;
    std::unordered_map<QueryId, PerQueryState> per_query;
    std::mutex mu;

    // loads
    bool loads_started = false;
    std::vector<LoadItem> loads;
    std::vector<Event> h2d_done, load_done;
    DevicePlan load_plan;
    size_t ring_slot_bytes = 0;
    bool loads_ce = false;        // lazy copy-engine pipeline in use
    bool loads_finalized = false;
    uint32_t next_load = 0;       // next layer to enqueue
    uint32_t load_depth = 1;
    size_t load_layer_bytes = 0;

    // stores
    bool stores_reserved = false;
    uint32_t next_store_layer = 0;
    std::vector<bool> store_done;
    bool stores_sealed = false, stores_waited = false;
    std::vector<StoreItem> stores;
    std::vector<Digest> store_touches;  // LRU touch order of the batch's puts (begin_write_batch)
    std::shared_ptr<ReleaseState> loads_released;  // set by the load release callback
    std::vector<Event> compute_done, gathered, d2h_done;
    Event store_complete;
    Event t0{true};  // timeline origin (recorded when loads are enqueued)
    DevicePlan store_plan;
    std::atomic<bool> committed{false};
    bool any_store_writes = false;
    bool store_ce = false;         // copy-engine store path for this batch
    uint32_t store_depth = 1;
    size_t store_layer_bytes = 0;  // one staging layer
    Connector::StagingRing* store_ring = nullptr;  // held until the stores are sealed

    ~BatchState() {
        // Device buffers above may still feed in-flight work: drain first.
        try {
            if (loads_ce && !loads_finalized) {  // engine stopped waiting early: finish the loads
                std::lock_guard io(conn->io_mu_);
                conn->enqueue_load_layers(*this, num_layers);
            }
            if (loads_started && !load_done.empty()) load_done.back().sync();
            if (any_store_writes) {
                // This batch's own completion only: later batches may already
                // be queued on the same streams.
                if (stores_sealed) {
                    store_complete.sync();  // recorded after the commit callback: `committed` is final
                } else {
                    TKV_CUDA(cudaStreamSynchronize(conn->store_stream_));
                    TKV_CUDA(cudaStreamSynchronize(conn->d2h_stream_));
                }
                if (!committed.load()) {
                    for (auto& s : stores)
                        if (s.w.kind == SlotWrite::Kind::write)
                            conn->store().commit_write(
                                plans[s.plan].store_plan[s.desc].key.digest,
                                Status{Errc::io_error, "batch dropped before stores finished"});
                }
            }
        } catch (...) {
        }
        if (store_ring != nullptr) {  // never sealed: the streams were drained above
            std::lock_guard io(conn->io_mu_);
            store_ring->owner = nullptr;
            store_ring->used = false;
        }
    }
};

}  // namespace detail

using detail::BatchState;

TransferMode ConnectorMetadata::mode() const {
    std::lock_guard lock(state_->mu);
    return state_->mode;
}
const std::vector<QueryPlan>& ConnectorMetadata::plans() const { return state_->plans; }
size_t ConnectorMetadata::loaded_tokens(QueryId id) const {
    std::lock_guard lock(state_->mu);
    auto it = state_->per_query.find(id);
    return it == state_->per_query.end() ? 0 : it->second.loaded;
}
std::vector<std::pair<ChunkKey, Status>> ConnectorMetadata::store_results(QueryId id) const {
    std::lock_guard lock(state_->mu);
    auto it = state_->per_query.find(id);
    if (it == state_->per_query.end()) return {};
    return it->second.store_results;
}

std::vector<float> ConnectorMetadata::timeline() const {
    const BatchState& b = *state_;
    std::vector<float> out(size_t(b.num_layers) * 5, -1.f);
    auto get = [&](const std::vector<Event>& v, uint32_t l) {
        return (b.loads_started && l < v.size()) ? elapsed(b.t0, v[l]) : -1.f;
    };
    for (uint32_t l = 0; l < b.num_layers; ++l) {
        out[5 * l + 0] = get(b.h2d_done, l);
        out[5 * l + 1] = get(b.load_done, l);
        out[5 * l + 2] = get(b.compute_done, l);
        out[5 * l + 3] = get(b.gathered, l);
        out[5 * l + 4] = get(b.d2h_done, l);
    }
    return out;
}

float ConnectorMetadata::origin_since(cudaEvent_t ref) const {
    float ms = -1.f;
    if (!state_->loads_started || cudaEventElapsedTime(&ms, ref, state_->t0) != cudaSuccess) {
        cudaGetLastError();
        return -1.f;
    }
    return ms;
}

Connector::Connector(TieredStore& store, PagedKVStore& pages, Config cfg)
    : store_(store),
      pages_(pages),
      cfg_(cfg),
      hasher_(store.config().model.model_tag, store.config().chunk_size, pages.device()) {
    TKV_CUDA(cudaSetDevice(pages_.device()));
    if (cfg_.staging_depth == 0) cfg_.staging_depth = 1;
    h2d_stream_ = Stream::create();
    load_stream_ = Stream::create();
    store_stream_ = Stream::create();
    d2h_stream_ = Stream::create();
    hasher_.enable_memo(cfg_.memo_entries);
    // The lookup kernels decide the stored prefix from a device mirror of the
    // tier's present set (TKV_NO_PRESENCE=1: the host index, A/B only).
    if (std::getenv("TKV_NO_PRESENCE") == nullptr) {
        const size_t id = store_.presence_subscribe();
        TieredStore* st = &store_;
        hasher_.enable_presence(store_.slab_slots(), [st, id](bool full, std::vector<std::pair<Digest, bool>>& out,
                                                             bool& reset) { st->presence_drain(id, full, out, reset); });
    }
}

Connector::Connector(TieredStore& store, PagedKVStore& pages) : Connector(store, pages, Config{}) {}

Connector::~Connector() {
    try {
        TKV_CUDA(cudaStreamSynchronize(h2d_stream_));
        TKV_CUDA(cudaStreamSynchronize(load_stream_));
        TKV_CUDA(cudaStreamSynchronize(store_stream_));
        TKV_CUDA(cudaStreamSynchronize(d2h_stream_));
    } catch (...) {
    }
}

// Prompt buffers of finished queries are kept and reused: they are mapped
// pinned memory (the lookup kernels read the prompt from the query state
// itself, no second staging copy), whose allocation and release are slow and
// can synchronize the device. Caller holds mu_.
size_t Connector::prompt_capacity(size_t n) {
    size_t c = 4096;
    while (c < n) c <<= 1;
    return c;
}

void Connector::recycle_prompt(PinnedTokens&& v) {
    if (v.capacity() == 0 || prompt_pool_.size() >= 256) return;
    v.clear();
    prompt_pool_.push_back(std::move(v));
}

void Connector::recycle_prompt_into(PinnedTokens& dst, size_t n) {
    for (size_t i = prompt_pool_.size(); i-- > 0;) {
        if (prompt_pool_[i].capacity() >= n) {
            recycle_prompt(std::move(dst));
            dst = std::move(prompt_pool_[i]);
            prompt_pool_.erase(prompt_pool_.begin() + std::ptrdiff_t(i));
            return;
        }
    }
}

const std::vector<ChunkKey>& Connector::keys_for(QueryState& qs, TokenSpanView prompt) {
    const size_t rows = (prompt.size() + store_.config().chunk_size - 1) / store_.config().chunk_size;
    // Recompute when the prompt differs or the lookup stopped at the first
    // absent chunk (the memo serves the part it already hashed).
    if (qs.keys.size() != rows || qs.prompt.size() != prompt.size() ||
        !std::equal(prompt.begin(), prompt.end(), qs.prompt.begin())) {
        if (qs.prompt.capacity() < prompt.size()) qs.prompt.reserve(prompt_capacity(prompt.size()));
        qs.prompt.resize(prompt.size());
        host_copy(qs.prompt.data(), prompt.data(), prompt.size() * sizeof(TokenId));
        qs.keys = chunk_keys(hasher_, prompt);
    }
    return qs.keys;
}

size_t Connector::get_num_new_matched_tokens(QueryId id, TokenSpanView prompt) {
    return get_num_new_matched_tokens(std::vector<QueryId>{id}, {prompt})[0];
}

std::vector<size_t> Connector::get_num_new_matched_tokens(
    const std::vector<QueryId>& ids, const std::vector<TokenSpanView>& prompts) {
    const size_t cs = store_.config().chunk_size;
    static const bool trace = std::getenv("TKV_TRACE_LOOKUP") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    size_t tokens = 0;
    for (const auto& p : prompts) tokens += p.size();
    if (tokens * sizeof(TokenId) >= (128u << 10)) host_copy_prime();  // the copies below are parallel
    // The query state keeps a copy of each prompt; it is made while the
    // lookup's first launch runs (pooled buffers, swapped in below).
    std::vector<PinnedTokens> staged(ids.size());
    std::vector<const TokenId*> mapped(ids.size());
    {
        std::lock_guard lock(mu_);
        for (size_t q = 0; q < ids.size(); ++q) {
            recycle_prompt_into(staged[q], prompts[q].size());
            // power-of-two capacity: prompts of varying length reuse pooled
            // buffers instead of allocating pinned memory (which waits for the
            // device) on the lookup path; assign() below keeps this buffer
            staged[q].reserve(prompt_capacity(prompts[q].size()));
            mapped[q] = staged[q].data();
        }
    }
    // LPM (tokens.cpp:59-69): the chain only as far as the first absent
    // chunk, like the reference's lookup; the leading present chunks are
    // probed under one store lock per query. Planning completes the chain.
    std::vector<size_t> present_rows;
    auto digests = hasher_.hash_prefix(
        prompts, [this](const std::vector<Digest>& d) { return store_.present_prefix(d); },
        [&] {
            for (size_t q = 0; q < ids.size(); ++q) {
                staged[q].resize(prompts[q].size());
                host_copy(staged[q].data(), prompts[q].data(), prompts[q].size() * sizeof(TokenId));
            }
        },
        &present_rows, &mapped);
    const auto t1 = std::chrono::steady_clock::now();
    std::vector<size_t> out(ids.size());
    for (size_t q = 0; q < ids.size(); ++q) {
        std::vector<ChunkKey> keys(digests[q].size());
        for (size_t i = 0; i < keys.size(); ++i)
            keys[i] = ChunkKey{digests[q][i], store_.config().model.model_tag, uint32_t(i)};
        const size_t n = prompts[q].size();
        const size_t present = present_rows[q];  // decided on the device (presence index) where it could
        const size_t lpm = present == 0 ? 0 : std::min(n, present * cs);
        const size_t cap = n == 0 ? 0 : n - 1;  // connector.cpp:75-76
        const size_t matched = std::min(lpm, cap);
        std::lock_guard lock(mu_);
        QueryState& qs = queries_[ids[q]];
        std::swap(qs.prompt, staged[q]);
        recycle_prompt(std::move(staged[q]));
        qs.keys = std::move(keys);
        qs.lpm = lpm;
        qs.matched = matched;
        out[q] = matched;
    }
    if (trace) {
        const auto t2 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[tkv lookup] hash=%.1fus lpm+state=%.1fus\n",
                     std::chrono::duration<double, std::micro>(t1 - t0).count(),
                     std::chrono::duration<double, std::micro>(t2 - t1).count());
    }
    return out;
}

Status Connector::update_state_after_alloc(QueryId id, size_t blocks, size_t num_external_blocks) {
    std::lock_guard lock(mu_);
    auto it = queries_.find(id);
    if (it == queries_.end()) return Status{Errc::invalid_argument, "unknown query"};
    const size_t pt = store_.config().model.page_tokens;
    const size_t needed = (it->second.matched + pt - 1) / pt;
    if (num_external_blocks != needed)
        return Status{Errc::invalid_argument, "external block count mismatch"};
    if (blocks < needed) return Status{Errc::invalid_argument, "inconsistent alloc"};
    it->second.blocks = blocks;
    return Status::success();
}

ConnectorMetadata Connector::build_connector_meta(const SchedulerOutput& out) {
    const auto& cfg = store_.config();
    auto b = std::make_shared<BatchState>();
    b->conn = this;
    b->mode = cfg_.mode;
    b->num_layers = cfg.model.num_layers;
    b->store_done.assign(b->num_layers, false);

    for (const auto& sq : out.queries) {
        QueryPlan plan;
        plan.id = sq.id;
        plan.prompt_tokens = sq.prompt.size();
        std::vector<ChunkKey> keys;
        size_t lpm = 0, matched = 0;
        {
            std::lock_guard lock(mu_);
            QueryState& qs = queries_[sq.id];
            keys = keys_for(qs, sq.prompt);  // cached from lookup: no re-hash
            lpm = qs.lpm;
            matched = qs.matched;
        }
        plan.matched_tokens = matched;
        const auto spans = chunk_tokens(sq.prompt.size(), cfg.chunk_size);
        // Load descriptors: stored chunking of the uncapped match, spans
        // clipped to the capped match (connector.cpp:136-147).
        for (size_t i = 0; i < spans.size() && spans[i].end <= lpm; ++i) {
            ChunkSpan span = spans[i];
            const uint32_t record_tokens = uint32_t(span.length());
            if (span.start >= matched) break;
            span.end = std::min(span.end, matched);
            plan.load_plan.push_back({keys[i], span, record_tokens});
        }
        // Store descriptors: chunks absent at build time (connector.cpp:100-110).
        std::vector<Digest> digests(keys.size());
        for (size_t i = 0; i < keys.size(); ++i) digests[i] = keys[i].digest;
        const std::vector<bool> present = store_.present_mask(digests);
        for (size_t i = 0; i < spans.size(); ++i) {
            if (present[i]) continue;
            plan.store_plan.push_back({keys[i], spans[i], uint32_t(spans[i].length())});
        }
        detail::PerQueryState pq;
        pq.loaded = matched;
        b->per_query.emplace(sq.id, std::move(pq));
        b->plans.push_back(std::move(plan));
    }
    ConnectorMetadata meta;
    meta.state_ = std::move(b);
    return meta;
}

// Size for a staging ring that must grow: at least `need`, and at least twice
// the current size up to the depth x budget bound, so batches of varying
// size stop reallocating (each growth synchronizes the ring's streams and
// calls cudaMalloc, which must not recur inside a serving loop).
size_t Connector::ring_growth(size_t need, size_t current, uint32_t depth) const {
    // Twice what is needed (a first reservation included): a later, larger
    // batch (config 2's waves) must not reallocate, since freeing the old ring
    // waits for every transfer in flight.
    const size_t cap = size_t(depth) * cfg_.staging_budget_bytes;
    return std::max(need, std::min(2 * std::max(current, need), cap));
}

// --- loads -----------------------------------------------------------------

Status Connector::enqueue_loads(BatchState& b) {
    const auto& model = store_.config().model;
    const uint32_t L = b.num_layers;
    const uint32_t pt = model.page_tokens;
    const size_t bpt = model.bytes_per_token_per_layer;

    // Safe prefix per query (connector.cpp:196-216): a chunk that vanished, a
    // record whose geometry differs from the plan, or pages that cannot take
    // the span end the deliverable prefix at that chunk.
    for (const auto& plan : b.plans) {
        size_t safe = plan.matched_tokens;
        for (const auto& d : plan.load_plan) {
            bool ok = true;
            for (uint32_t l = 0; l < L && ok; ++l)
                ok = pages_.check_writable_span(plan.id, l, d.span.start / pt, d.span.length()).ok();
            Result<SlotRead> r = ok ? store_.acquire(d.key.digest, d.record_tokens)
                                    : Result<SlotRead>(Status{Errc::size_mismatch, "pages"});
            if (!r.ok()) {
                safe = d.span.start;
                break;
            }
            b.loads.push_back({plan.id, d.key.digest, r.value(), d.span, d.record_tokens, 0});
        }
        std::lock_guard lock(b.mu);
        auto& pq = b.per_query.at(plan.id);
        pq.loaded = std::min(pq.loaded, safe);
    }

    size_t layer_bytes = 0;
    for (auto& it : b.loads) {
        it.staging_off = layer_bytes;
        layer_bytes += ((it.span.length() * bpt + 255) / 256) * 256;
    }
    const bool blocking = b.mode == TransferMode::blocking;
    const bool zero_copy = blocking || cfg_.load_path == LoadPath::zero_copy;
    make_events(b.h2d_done, L);
    make_events(b.load_done, L);
    b.t0.record(h2d_stream_);
    b.loads_started = true;
    if (b.loads.empty()) {
        for (uint32_t l = 0; l < L; ++l) b.load_done[l].record(load_stream_);
        return Status::success();
    }

    // Device page tables, then the copy plan (ordered on the load stream).
    std::unordered_map<QueryId, PagedKVStore::DeviceTable> tables;
    for (const auto& it : b.loads) {
        if (tables.count(it.id)) continue;
        auto t = pages_.device_table(it.id, load_stream_);
        if (!t.ok()) return t.status();
        tables.emplace(it.id, t.value());
    }
    const uint32_t depth = std::min<uint32_t>(cfg_.staging_depth, L);
    std::vector<std::vector<XferDesc>> vars(zero_copy ? 1 : depth);
    if (!zero_copy) {
        b.ring_slot_bytes = layer_bytes;
        // One load ring: an earlier batch still holding it (its engine has
        // not waited on every layer yet) enqueues its remaining layers first,
        // so no two batches ever interleave in the ring.
        if (load_ring_.owner != nullptr && load_ring_.owner != &b)
            enqueue_load_layers(*load_ring_.owner, load_ring_.owner->num_layers);
        if (size_t(depth) * layer_bytes > load_ring_.buf.bytes) {
            // every earlier batch has enqueued all its layers: once the ring's
            // last use finished, nothing reads the old buffer any more
            if (load_ring_.used) load_ring_.free.sync();
            load_ring_.buf.reserve(ring_growth(size_t(depth) * layer_bytes, load_ring_.buf.bytes, depth));
        }
        staging_peak_ = std::max(staging_peak_, size_t(depth) * layer_bytes);
    }
    for (size_t v = 0; v < vars.size(); ++v) {
        for (const auto& it : b.loads) {
            XferDesc d;
            const auto& t = tables.at(it.id);
            d.table = t.ptr;
            d.table_stride = t.stride;
            d.first_page = uint32_t(it.span.start / pt);
            d.n_tokens = uint32_t(it.span.length());
            if (zero_copy) {
                d.chunk = reinterpret_cast<uint64_t>(it.slot.dev);
                d.layer_stride = uint64_t(it.record_tokens) * bpt;
            } else {
                d.chunk = reinterpret_cast<uint64_t>(load_ring_.buf.ptr + v * layer_bytes + it.staging_off);
                d.layer_stride = 0;
            }
            vars[v].push_back(d);
        }
    }
    b.load_plan.build(plan_pool_, vars, pt, pages_.page_bytes(), L, load_stream_);
    const PagedLayout layout = pages_.layout();

    if (zero_copy && blocking) {
        TKV_CUDA(launch_paged_copy(layout, b.load_plan.plan(0, 0, L), CopyDir::scatter,
                                   cfg_.load_ctas, load_stream_));
        for (uint32_t l = 0; l < L; ++l) b.load_done[l].record(load_stream_);
    } else if (zero_copy) {
        for (uint32_t l = 0; l < L; ++l) {
            TKV_CUDA(launch_paged_copy(layout, b.load_plan.plan(0, l, 1), CopyDir::scatter,
                                       cfg_.load_ctas, load_stream_));
            b.load_done[l].record(load_stream_);
        }
    } else {
        // Layerwise copy-engine pipeline through a `depth`-layer staging ring,
        // enqueued lazily `depth` layers ahead of the engine (the reference
        // launches layer l+1 when the engine waits for l, connector.cpp:268-279):
        // the copy engines are shared with the engine's own transfers, which
        // must not queue behind a whole prompt of loads.
        if (load_ring_.used) load_ring_.free.wait_on(h2d_stream_);  // previous batch done with the ring
        load_ring_.owner = &b;
        b.loads_ce = true;
        b.load_depth = depth;
        b.load_layer_bytes = layer_bytes;
        b.next_load = 0;
        enqueue_load_layers(b, std::min<uint32_t>(L, depth + 1));
    }
    // Pages hold the bytes once the stream reaches them; the slots are free
    // for eviction after the last scatter.
    for (const auto& it : b.loads)
        for (uint32_t l = 0; l < L; ++l)
            pages_.mark_span_populated(it.id, l, it.span.start / pt, it.span.length());
    if (!b.loads_ce) {  // the lazy CE pipeline releases after its last layer
        b.loads_released = std::make_shared<ReleaseState>();
        auto* ctx = new ReleaseCtx{&store_, {}, b.loads_released};
        for (const auto& it : b.loads) ctx->digests.push_back(it.digest);
        TKV_CUDA(cudaLaunchHostFunc(load_stream_, release_cb, ctx));
    }
    if (blocking) TKV_CUDA(cudaStreamSynchronize(load_stream_));
    return Status::success();
}

void Connector::enqueue_load_layers(BatchState& b, uint32_t upto) {
    if (!b.loads_ce) return;
    const auto& model = store_.config().model;
    const size_t bpt = model.bytes_per_token_per_layer;
    const PagedLayout layout = pages_.layout();
    const size_t n = b.loads.size();
    std::vector<void*> dst(n);
    std::vector<const void*> src(n);
    std::vector<size_t> sizes(n);
    upto = std::min(upto, b.num_layers);
    for (uint32_t l = b.next_load; l < upto; ++l) {
        const uint32_t r = l % b.load_depth;
        if (l >= b.load_depth) b.load_done[l - b.load_depth].wait_on(h2d_stream_);
        for (size_t i = 0; i < n; ++i) {
            const auto& it = b.loads[i];
            src[i] = it.slot.host + size_t(l) * it.record_tokens * bpt;
            dst[i] = load_ring_.buf.ptr + size_t(r) * b.load_layer_bytes + it.staging_off;
            sizes[i] = it.span.length() * bpt;
        }
        TKV_CUDA(ce_copy_pieces(dst.data(), src.data(), sizes.data(), n, cudaMemcpyHostToDevice,
                                h2d_stream_, &copy_stats_));
        b.h2d_done[l].record(h2d_stream_);
        b.h2d_done[l].wait_on(load_stream_);
        TKV_CUDA(launch_paged_copy(layout, b.load_plan.plan(r, l, 1), CopyDir::scatter,
                                   cfg_.load_ctas, load_stream_));
        b.load_done[l].record(load_stream_);
    }
    if (upto > b.next_load) b.next_load = upto;
    if (b.next_load == b.num_layers && !b.loads_finalized) {
        b.loads_finalized = true;
        load_ring_.free.record(load_stream_);
        load_ring_.used = true;
        load_ring_.owner = nullptr;
        b.loads_released = std::make_shared<ReleaseState>();
        auto* ctx = new ReleaseCtx{&store_, {}, b.loads_released};
        for (const auto& it : b.loads) ctx->digests.push_back(it.digest);
        TKV_CUDA(cudaLaunchHostFunc(load_stream_, release_cb, ctx));
    }
}

Status Connector::start_load_kv(ConnectorMetadata& meta) {
    if (!meta) return Status{Errc::invalid_argument, "empty metadata"};
    BatchState& b = *meta.state_;
    std::lock_guard io(io_mu_);
    if (b.loads_started) return Status::success();
    const size_t bpt = store_.config().model.bytes_per_token_per_layer;
    size_t layer_bytes = 0;
    for (const auto& plan : b.plans)
        for (const auto& d : plan.load_plan) layer_bytes += d.span.length() * bpt;
    if (layer_bytes > cfg_.staging_budget_bytes) {  // connector.cpp:244-256
        std::lock_guard lock(b.mu);
        b.mode = TransferMode::blocking;
    }
    try {
        return enqueue_loads(b);
    } catch (const CudaError& e) {
        return Status{Errc::cuda_error, e.what()};
    }
}

Status Connector::wait_load_kv(ConnectorMetadata& meta, uint32_t layer) {
    if (!meta) return Status{Errc::invalid_argument, "empty metadata"};
    BatchState& b = *meta.state_;
    if (layer >= b.num_layers) return Status{Errc::invalid_argument, "layer out of range"};
    if (!b.loads_started) {
        Status st = start_load_kv(meta);
        if (!st.ok()) return st;
    }
    try {
        if (b.loads_ce && b.next_load < b.num_layers) {
            std::lock_guard io(io_mu_);
            enqueue_load_layers(b, layer + 2 + b.load_depth);  // keep `depth` layers in flight
        }
        b.load_done[layer].wait_on(cfg_.engine_stream);  // engine stream, not the host, waits
    } catch (const CudaError& e) {
        return Status{Errc::cuda_error, e.what()};
    }
    return Status::success();
}

// --- stores ----------------------------------------------------------------

Status Connector::reserve_stores(BatchState& b) {
    const auto& model = store_.config().model;
    const uint32_t pt = model.page_tokens;
    const size_t bpt = model.bytes_per_token_per_layer;
    std::vector<XferDesc> descs;
    std::unordered_map<QueryId, PagedKVStore::DeviceTable> tables;
    // Every slot of the batch in one reservation, in the reference's
    // batch_put order (plans, then chunks), with its eviction outcome.
    std::vector<TieredStore::WriteSpec> specs;
    for (const auto& plan : b.plans)
        for (const auto& d : plan.store_plan) specs.push_back({d.key.digest, d.record_tokens, cfg_.pin_stores});
    std::unordered_map<Digest, uint32_t, DigestHasher> own_shares;
    for (const auto& it : b.loads) ++own_shares[it.digest];
    auto writes = store_.begin_write_batch(specs, own_shares, &b.store_touches);
    size_t k = 0;
    for (size_t p = 0; p < b.plans.size(); ++p) {
        const auto& plan = b.plans[p];
        for (size_t i = 0; i < plan.store_plan.size(); ++i) {
            const auto& d = plan.store_plan[i];
            detail::StoreItem item{p, i, Status::success(), {}};
            auto& w = writes[k++];
            if (!w.ok()) {
                item.status = w.status();
            } else {
                item.w = w.value();
                if (item.w.kind == SlotWrite::Kind::write) {
                    if (!tables.count(plan.id)) {
                        auto t = pages_.device_table(plan.id, store_stream_);
                        if (!t.ok()) return t.status();
                        tables.emplace(plan.id, t.value());
                    }
                    XferDesc x;
                    x.chunk = reinterpret_cast<uint64_t>(item.w.dev);
                    x.layer_stride = uint64_t(d.record_tokens) * bpt;
                    x.table = tables.at(plan.id).ptr;
                    x.table_stride = tables.at(plan.id).stride;
                    x.first_page = uint32_t(d.span.start / pt);
                    x.n_tokens = uint32_t(d.span.length());
                    descs.push_back(x);
                }
            }
            b.stores.push_back(std::move(item));
        }
    }
    b.any_store_writes = !descs.empty();
    make_events(b.compute_done, b.num_layers);
    b.stores_reserved = true;
    // Copy-engine path (layerwise only): K1 writes one layer of every chunk
    // into an HBM staging ring slot; the CE then copies each chunk-layer
    // slice into its pinned slot at offset layer*T*bpt (store.cpp:343-345).
    b.store_ce = cfg_.store_path == StorePath::copy_engine &&
                 b.mode == TransferMode::layerwise && b.any_store_writes;
    if (!b.store_ce) {
        b.store_plan.build(plan_pool_, {descs}, pt, pages_.page_bytes(), b.num_layers, store_stream_);
        return Status::success();
    }
    size_t off = 0;
    for (auto& s : b.stores) {
        if (s.w.kind != SlotWrite::Kind::write) continue;
        const auto& d = b.plans[s.plan].store_plan[s.desc];
        s.staging_off = off;
        s.rows = d.span.length();
        s.record_tokens = d.record_tokens;
        off += ((s.rows * bpt + 255) / 256) * 256;
    }
    b.store_layer_bytes = off;
    b.store_depth = std::min<uint32_t>(std::max<uint32_t>(cfg_.staging_depth, 1), b.num_layers);
    const size_t need = size_t(b.store_depth) * off;
    StagingRing* ring = acquire_store_ring(b, need, b.store_depth);
    staging_peak_ = std::max(staging_peak_, need);
    std::vector<std::vector<XferDesc>> vars(b.store_depth, descs);
    for (uint32_t r = 0; r < b.store_depth; ++r) {
        size_t k = 0;
        for (const auto& s : b.stores) {
            if (s.w.kind != SlotWrite::Kind::write) continue;
            vars[r][k].chunk = reinterpret_cast<uint64_t>(ring->buf.ptr + r * off + s.staging_off);
            vars[r][k].layer_stride = 0;
            ++k;
        }
    }
    b.store_plan.build(plan_pool_, vars, pt, pages_.page_bytes(), b.num_layers, store_stream_);
    make_events(b.gathered, b.num_layers);
    make_events(b.d2h_done, b.num_layers);
    if (ring->used) ring->free.wait_on(store_stream_);  // the ring's previous batch finished its copies
    return Status::success();
}

// A store ring for batch b: a free one large enough, else a free one grown
// (after its last use finished), else a new one. A ring stays with its batch
// until the batch's last layer is enqueued (start_store_kv seals it), so two
// batches whose stores overlap never share one. Caller holds io_mu_.
Connector::StagingRing* Connector::acquire_store_ring(BatchState& b, size_t need, uint32_t depth) {
    StagingRing* pick = nullptr;
    for (auto& r : store_rings_)
        if (r->owner == nullptr && r->buf.bytes >= need) {
            pick = r.get();
            break;
        }
    if (pick == nullptr) {
        for (auto& r : store_rings_)
            if (r->owner == nullptr) {
                pick = r.get();
                break;
            }
        if (pick == nullptr) {
            store_rings_.push_back(std::make_unique<StagingRing>());
            pick = store_rings_.back().get();
        }
        if (pick->used) pick->free.sync();  // its last batch's copies have finished
        pick->buf.reserve(ring_growth(need, pick->buf.bytes, depth));
    }
    pick->owner = &b;
    b.store_ring = pick;
    return pick;
}

Status Connector::store_layers(BatchState& b, uint32_t first, uint32_t last) {
    const auto& model = store_.config().model;
    const uint32_t pt = model.page_tokens;
    // Gather readability (check_readable, paged_store.cpp:94-111) per layer.
    for (uint32_t l = first; l < last; ++l)
        for (const auto& s : b.stores) {
            if (s.w.kind != SlotWrite::Kind::write) continue;
            const auto& plan = b.plans[s.plan];
            const auto& d = plan.store_plan[s.desc];
            Status st = pages_.check_readable_span(plan.id, l, d.span.start / pt, d.span.length());
            if (!st.ok()) return st;
        }
    if (b.store_plan.n_desc == 0) return Status::success();
    const PagedLayout layout = pages_.layout();
    // K1 for these layers, ordered after the engine's compute of them.
    b.compute_done[first].record(cfg_.engine_stream);
    b.compute_done[first].wait_on(store_stream_);
    // ... and after this batch's own loads of them: a slot this batch evicts
    // may be one it is still loading (begin_write_batch), and layer l of the
    // new chunk must not land before layer l of the old one was read. An
    // engine that waited on wait_load_kv(l) before computing l already
    // implies this; one that did not (or a lazy pipeline not yet enqueued
    // that far) gets the order here.
    if (b.loads_started && !b.loads.empty()) {
        if (b.loads_ce && b.next_load < last) enqueue_load_layers(b, last);
        b.load_done[last - 1].wait_on(store_stream_);
    }
    if (!b.store_ce) {
        TKV_CUDA(launch_paged_copy(layout, b.store_plan.plan(0, first, last - first),
                                   CopyDir::gather, cfg_.store_ctas, store_stream_));
        return Status::success();
    }
    const size_t bpt = model.bytes_per_token_per_layer;
    for (uint32_t l = first; l < last; ++l) {
        const uint32_t r = l % b.store_depth;
        if (l >= b.store_depth) b.d2h_done[l - b.store_depth].wait_on(store_stream_);
        TKV_CUDA(launch_paged_copy(layout, b.store_plan.plan(r, l, 1), CopyDir::gather,
                                   cfg_.load_ctas, store_stream_));
        b.gathered[l].record(store_stream_);
        b.gathered[l].wait_on(d2h_stream_);
        std::vector<void*> dst;
        std::vector<const void*> src;
        std::vector<size_t> sizes;
        for (const auto& s : b.stores) {
            if (s.w.kind != SlotWrite::Kind::write) continue;
            dst.push_back(s.w.host + size_t(l) * s.record_tokens * bpt);
            src.push_back(b.store_ring->buf.ptr + size_t(r) * b.store_layer_bytes + s.staging_off);
            sizes.push_back(s.rows * bpt);
        }
        TKV_CUDA(ce_copy_pieces(dst.data(), src.data(), sizes.data(), dst.size(),
                                cudaMemcpyDeviceToHost, d2h_stream_, &copy_stats_));
        b.d2h_done[l].record(d2h_stream_);
    }
    return Status::success();
}

Status Connector::start_store_kv(ConnectorMetadata& meta) {
    if (!meta) return Status{Errc::invalid_argument, "empty metadata"};
    BatchState& b = *meta.state_;
    uint32_t first = 0, last = 0;
    {
        std::lock_guard lock(b.mu);
        if (b.mode == TransferMode::blocking) {
            first = 0;
            last = b.num_layers;
            b.next_store_layer = b.num_layers;
        } else {
            if (b.next_store_layer >= b.num_layers) return Status::success();
            first = b.next_store_layer;
            last = ++b.next_store_layer;
        }
    }
    try {
        std::lock_guard io(io_mu_);
        if (!b.stores_reserved) {
            Status st = reserve_stores(b);
            if (!st.ok()) return st;
        }
        Status st = store_layers(b, first, last);
        if (!st.ok()) return st;
        {
            std::lock_guard lock(b.mu);
            for (uint32_t l = first; l < last; ++l) b.store_done[l] = true;
        }
        if (last == b.num_layers && !b.stores_sealed) {
            b.stores_sealed = true;
            cudaStream_t done_stream = b.store_ce ? d2h_stream_.s : store_stream_.s;
            if (b.store_ring != nullptr) {
                b.store_ring->free.record(d2h_stream_);
                b.store_ring->used = true;
                b.store_ring->owner = nullptr;
                b.store_ring = nullptr;
            }
            if (b.any_store_writes) {
                auto* ctx = new CommitCtx{&store_, {}, &b.committed, std::move(b.store_touches)};
                for (const auto& s : b.stores)
                    if (s.w.kind == SlotWrite::Kind::write)
                        ctx->digests.push_back(b.plans[s.plan].store_plan[s.desc].key.digest);
                TKV_CUDA(cudaLaunchHostFunc(done_stream, commit_cb, ctx));
            } else {
                b.committed.store(true);
            }
            // Recorded after the commit callback: a stream does not pass a host
            // function until it returned, so whoever syncs this event (the
            // final wait, ~BatchState) sees the batch committed and the
            // callback done with the batch's memory.
            b.store_complete.record(done_stream);
        }
    } catch (const CudaError& e) {
        return Status{Errc::cuda_error, e.what()};
    }
    if (b.mode == TransferMode::blocking) return wait_store_kv(meta, b.num_layers - 1);
    return Status::success();
}

Status Connector::wait_store_kv(ConnectorMetadata& meta, uint32_t layer) {
    if (!meta) return Status{Errc::invalid_argument, "empty metadata"};
    BatchState& b = *meta.state_;
    if (layer >= b.num_layers) return Status{Errc::invalid_argument, "layer out of range"};
    {
        std::lock_guard lock(b.mu);
        if (!b.store_done[layer]) return Status{Errc::invalid_argument, "store for layer not started"};
        if (layer + 1 < b.num_layers || b.stores_waited) return Status::success();
    }
    // Final wait: the bytes landed, then per-chunk statuses (connector.cpp:372-391).
    try {
        b.store_complete.sync();
    } catch (const CudaError& e) {
        return Status{Errc::cuda_error, e.what()};
    }
    // The reference's loads have released their shares by the time its
    // stores are sealed; so do ours by the time this returns (the next
    // batch's slot reservation must see the same evictable set).
    if (b.loads_released) b.loads_released->wait();
    std::unordered_map<QueryId, std::vector<std::pair<ChunkKey, Status>>> results;
    for (auto& s : b.stores) {
        const auto& plan = b.plans[s.plan];
        Status st = s.status.ok() ? s.w.handle.wait() : s.status;
        results[plan.id].emplace_back(plan.store_plan[s.desc].key, st);
    }
    std::lock_guard lock(b.mu);
    for (auto& [id, r] : results) b.per_query.at(id).store_results = std::move(r);
    b.stores_waited = true;
    return Status::success();
}

// --- decode ----------------------------------------------------------------

Status Connector::begin_decode(QueryId id) {
    std::lock_guard lock(mu_);
    auto it = queries_.find(id);
    if (it == queries_.end() || it->second.prompt.empty())
        return Status{Errc::invalid_argument, "no planned query"};
    QueryState& qs = it->second;
    if (qs.decode) return Status{Errc::duplicate_key, "decode already open"};
    const size_t cs = store_.config().chunk_size;
    const auto& keys = keys_for(qs, qs.prompt);
    const size_t full = qs.prompt.size() / cs;
    auto ds = std::make_unique<DecodeState>(DecodeState{KeyChain(hasher_), {}, full * cs, {}, {}});
    if (full > 0) ds->chain.reset(keys[full - 1].digest, uint32_t(full));
    ds->tokens.assign(qs.prompt.begin() + full * cs, qs.prompt.end());
    qs.decode = std::move(ds);
    return Status::success();
}

Status Connector::flush_decode(QueryId id, QueryState& qs) {
    DecodeState& ds = *qs.decode;
    if (ds.tokens.empty()) return Status::success();
    const auto& model = store_.config().model;
    const uint32_t pt = model.page_tokens;
    const size_t n = ds.tokens.size();
    // Nothing changes (chain, buffered tokens, tier) unless the flush goes
    // through: the readability checks run first, the chain advances last.
    for (uint32_t l = 0; l < model.num_layers; ++l) {
        Status st = pages_.check_readable_span(id, l, ds.chunk_start / pt, n);
        if (!st.ok()) return st;
    }
    KeyChain chain = ds.chain;
    ChunkKey key = chain.next(ds.tokens);
    key.model_tag = model.model_tag;
    auto w = store_.begin_write(key.digest, uint32_t(n), cfg_.pin_stores);
    if (!w.ok()) {
        ds.puts.push_back(PutHandle::immediate(w.status()));
    } else if (w.value().kind != SlotWrite::Kind::write) {
        ds.puts.push_back(w.value().handle);
    } else {
        std::lock_guard io(io_mu_);
        auto t = pages_.device_table(id, store_stream_);
        if (!t.ok()) {
            store_.commit_write(key.digest, t.status());  // drop the claim
            return t.status();
        }
        XferDesc x;
        x.chunk = reinterpret_cast<uint64_t>(w.value().dev);
        x.layer_stride = uint64_t(n) * model.bytes_per_token_per_layer;
        x.table = t.value().ptr;
        x.table_stride = t.value().stride;
        x.first_page = uint32_t(ds.chunk_start / pt);
        x.n_tokens = uint32_t(n);
        auto plan = std::make_shared<DevicePlan>();
            plan->build(plan_pool_, {{x}}, pt, pages_.page_bytes(), model.num_layers, store_stream_);
        Event computed;
        computed.record(cfg_.engine_stream);
        computed.wait_on(store_stream_);
        TKV_CUDA(launch_paged_copy(pages_.layout(), plan->plan(0, 0, model.num_layers),
                                   CopyDir::gather, cfg_.store_ctas, store_stream_));
        // Asynchronous: the commit callback marks the chunk present and frees
        // the plan after the gather ran; finish_query waits on the handle.
        auto* ctx = new CommitCtx{&store_, {key.digest}, nullptr, {}, plan};
        TKV_CUDA(cudaLaunchHostFunc(store_stream_, commit_cb, ctx));
        ds.puts.push_back(w.value().handle);
    }
    ds.chain = chain;
    ds.flushed.push_back(key);
    ds.chunk_start += n;
    ds.tokens.clear();
    return Status::success();
}

Status Connector::append_decode(QueryId id, TokenId token) {
    std::lock_guard lock(mu_);
    auto it = queries_.find(id);
    if (it == queries_.end() || !it->second.decode)
        return Status{Errc::unknown_query, "decode not open"};
    DecodeState& ds = *it->second.decode;
    ds.tokens.push_back(token);
    if (ds.tokens.size() == store_.config().chunk_size) {
        Status st;
        try {
            st = flush_decode(id, it->second);
        } catch (const CudaError& e) {
            st = Status{Errc::cuda_error, e.what()};
        } catch (const std::exception& e) {
            st = Status{Errc::invalid_argument, e.what()};
        }
        // A chunk that could not be flushed (its KV not written yet) rejects
        // this append: the token is not taken, the buffer stays one short of
        // a chunk, and the engine may append it again.
        if (!st.ok()) ds.tokens.pop_back();
        return st;
    }
    return Status::success();
}

void Connector::append_decode_batch(const QueryId* ids, const TokenId* tokens, size_t n, Status* statuses) {
    for (size_t i = 0; i < n; ++i) statuses[i] = append_decode(ids[i], tokens[i]);
}

Result<std::vector<ChunkKey>> Connector::finish_query(QueryId id) {
    std::vector<ChunkKey> keys;
    std::unique_ptr<DecodeState> ds;
    {
        std::lock_guard lock(mu_);
        auto it = queries_.find(id);
        if (it != queries_.end() && it->second.decode) {
            try {
                Status st = flush_decode(id, it->second);
                if (!st.ok()) return st;
            } catch (const CudaError& e) {
                return Status{Errc::cuda_error, e.what()};
            } catch (const std::exception& e) {
                return Status{Errc::invalid_argument, e.what()};
            }
            ds = std::move(it->second.decode);
        }
        if (it != queries_.end()) {
            recycle_prompt(std::move(it->second.prompt));
            queries_.erase(it);
        }
    }
    if (ds) {
        for (const auto& h : ds->puts) h.wait();
        keys = std::move(ds->flushed);
    }
    return keys;
}

}  // namespace tkv
