// Engine-facing connector (mirror of include/tierkv/connector.hpp:14-152):
// the seven scheduler/worker calls (get_num_new_matched_tokens,
// update_state_after_alloc, build_connector_meta, start/wait_load_kv,
// start/wait_store_kv) plus decode storing and prefetch, with the
// reference's names, argument meaning and error behaviour.
//
// What changes is the execution model. The reference runs every byte on host
// threads: a TaskPool task per layer for loads (connector.cpp:179-237) and
// inline memcpys plus a record encode per chunk for stores (:281-358). Here
//   * lookup hashes each prompt once on the GPU (K3, with the prefix memo)
//     and caches the keys for planning;
//   * loads (copy-engine path, default): per layer one batched H2D of every
//     chunk-layer slice from the pinned slots into a device staging ring,
//     then one K2 scatter launch into the pages, enqueued a `staging_depth`
//     window ahead of the engine; wait_load_kv(l) makes the engine stream
//     wait on layer l's event instead of blocking the host;
//   * stores (copy-engine path, default): per layer K1 on a side stream,
//     ordered after the engine's compute of that layer, gathers every chunk
//     into an HBM staging ring and one batched D2H copies the slices into
//     their pinned slots; a stream callback marks the chunks present after
//     the last layer landed. Slots are claimed up front with the outcome of
//     the reference's sequential batch_put (TieredStore::begin_write_batch);
//   * zero-copy variants (K2 reading / K1 writing the pinned slots directly)
//     are selectable per connector.
// Blocking mode (configured, or a batch whose one-layer staging exceeds the
// budget, connector.cpp:244-256) moves all layers in one launch and returns
// only after the bytes are in place, like the reference.
#pragma once

#include <atomic>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "ce_copy.hpp"
#include "common.hpp"
#include "paged_store.hpp"
#include "store.hpp"
#include "tokens.hpp"

namespace tkv {

enum class TransferMode : uint8_t { layerwise, blocking };
enum class LoadPath : uint8_t { copy_engine, zero_copy };
// copy_engine: K1 into an HBM staging ring, then one batched CE D2H per layer.
// zero_copy:   K1 writes straight into the pinned slots over PCIe.
enum class StorePath : uint8_t { copy_engine, zero_copy };

struct ChunkDescriptor {
    ChunkKey key;
    ChunkSpan span;
    uint32_t record_tokens = 0;
};

struct ScheduledQuery {
    QueryId id = 0;
    std::vector<TokenId> prompt;
};

struct SchedulerOutput {
    std::vector<ScheduledQuery> queries;
};

struct QueryPlan {
    QueryId id = 0;
    size_t prompt_tokens = 0;
    size_t matched_tokens = 0;
    std::vector<ChunkDescriptor> load_plan;
    std::vector<ChunkDescriptor> store_plan;
};

namespace detail {
struct BatchState;
}

class ConnectorMetadata {
public:
    ConnectorMetadata() = default;
    TransferMode mode() const;
    const std::vector<QueryPlan>& plans() const;
    size_t loaded_tokens(QueryId id) const;
    std::vector<std::pair<ChunkKey, Status>> store_results(QueryId id) const;
    // Device timeline after completion: per layer, ms since loads were
    // enqueued for {h2d done, load done, compute done, gathered, d2h done}
    // (-1 where the event was not used). Diagnostics only.
    std::vector<float> timeline() const;
    // ms from a caller's (completed, timing) CUDA event to this batch's
    // timeline origin; places batches of a pipelined schedule on one axis.
    float origin_since(cudaEvent_t ref) const;
    explicit operator bool() const { return state_ != nullptr; }

private:
    friend class Connector;
    std::shared_ptr<detail::BatchState> state_;
};

class Connector {
public:
    struct Config {
        TransferMode mode = TransferMode::layerwise;
        bool pin_stores = false;
        // One layer of load bytes must fit, else the batch degrades to blocking.
        size_t staging_budget_bytes = 64ull << 20;
        uint32_t staging_depth = 2;      // layers of device staging in flight
        LoadPath load_path = LoadPath::copy_engine;
        StorePath store_path = StorePath::copy_engine;
        int store_ctas = 64;             // zero-copy K1 grid (PCIe-bound)
        int load_ctas = 0;               // K2 grid (0 = 2 x SMs)
        cudaStream_t engine_stream = nullptr;
        size_t memo_entries = 65536;     // prefix-digest memo links on the device (0 = off)
    };

    Connector(TieredStore& store, PagedKVStore& pages, Config cfg);
    Connector(TieredStore& store, PagedKVStore& pages);
    ~Connector();
    Connector(const Connector&) = delete;
    Connector& operator=(const Connector&) = delete;

    size_t get_num_new_matched_tokens(QueryId id, TokenSpanView prompt);
    // Batched lookup: one K3 launch for every prompt (extension).
    std::vector<size_t> get_num_new_matched_tokens(const std::vector<QueryId>& ids,
                                                   const std::vector<TokenSpanView>& prompts);
    Status update_state_after_alloc(QueryId id, size_t blocks, size_t num_external_blocks);
    ConnectorMetadata build_connector_meta(const SchedulerOutput& out);
    Status start_load_kv(ConnectorMetadata& meta);
    Status wait_load_kv(ConnectorMetadata& meta, uint32_t layer);
    Status start_store_kv(ConnectorMetadata& meta);
    Status wait_store_kv(ConnectorMetadata& meta, uint32_t layer);

    // Prefetch (connector.cpp:393-431) promotes matched chunks that sit only
    // in slower tiers (disk, remote) into the prefetch tiers. The pinned RAM
    // tier is the only tier on this path, so every present chunk is already
    // in the fastest one and both calls have nothing to do — kept so the API
    // is the reference's.
    void prefetch(TokenSpanView) {}
    void drain_prefetch() {}

    // Delayed decode storing (connector.cpp:434-497): the decode tokens' KV
    // lives in the query's pages; full chunks are gathered straight from the
    // pages into pinned slots (K1) as they complete.
    Status begin_decode(QueryId id);
    Status append_decode(QueryId id, TokenId token);
    // One generated token for each of many decoding queries (an engine's
    // decode step), one call; statuses[i] is append_decode's result.
    void append_decode_batch(const QueryId* ids, const TokenId* tokens, size_t n, Status* statuses);
    Result<std::vector<ChunkKey>> finish_query(QueryId id);

    const Config& config() const { return cfg_; }
    // Several batches may be in flight at once (a serving loop begins batch
    // k+1 before batch k's final wait_store_kv). The load staging ring is
    // held by one batch at a time: a batch that needs it while an earlier
    // one still has layers to enqueue first enqueues the earlier batch's
    // remaining layers. Store staging comes from a pool of rings, one per
    // batch whose stores are not yet sealed (normally one).
    TieredStore& store() { return store_; }
    PagedKVStore& pages() { return pages_; }
    KeyHasher& hasher() { return hasher_; }
    // Device staging high-water mark (bytes) across batches.
    size_t staging_peak_bytes() const { return staging_peak_; }
    // Host-tier copy-engine pieces and the copies they went out as (ce_copy.hpp).
    CopyRunStats copy_stats() {
        std::lock_guard io(io_mu_);
        return copy_stats_;
    }

private:
    friend struct detail::BatchState;
    struct DecodeState {
        KeyChain chain;
        std::vector<TokenId> tokens;   // tokens of the open (partial) chunk
        size_t chunk_start = 0;        // absolute position of tokens[0]
        std::vector<PutHandle> puts;
        std::vector<ChunkKey> flushed;
    };
    struct QueryState {
        PinnedTokens prompt;  // mapped pinned: the lookup kernels read it in place
        std::vector<ChunkKey> keys;  // chain of the whole prompt, hashed once
        size_t lpm = 0;
        size_t matched = 0;
        size_t blocks = 0;
        std::unique_ptr<DecodeState> decode;
    };

    const std::vector<ChunkKey>& keys_for(QueryState& qs, TokenSpanView prompt);
    size_t ring_growth(size_t need, size_t current, uint32_t depth) const;
    static size_t prompt_capacity(size_t n);  // pooled prompt buffers: power-of-two tokens
    void recycle_prompt(PinnedTokens&& v);
    void recycle_prompt_into(PinnedTokens& dst, size_t n);
    std::vector<PinnedTokens> prompt_pool_;  // guarded by mu_
    Status enqueue_loads(detail::BatchState& b);
    void enqueue_load_layers(detail::BatchState& b, uint32_t upto);
    Status store_layers(detail::BatchState& b, uint32_t first, uint32_t last);
    Status reserve_stores(detail::BatchState& b);
    Status flush_decode(QueryId id, QueryState& qs);

    TieredStore& store_;
    PagedKVStore& pages_;
    Config cfg_;
    KeyHasher hasher_;
    DualPool plan_pool_;  // per-batch launch plans (outlives every BatchState)
    Stream h2d_stream_, load_stream_, store_stream_, d2h_stream_;
    // A device staging ring; `owner` is the batch still enqueueing into it,
    // `free` (valid once `used`) marks the end of the last owner's device use.
    struct StagingRing {
        DeviceBuffer buf;
        Event free;
        bool used = false;
        detail::BatchState* owner = nullptr;
    };
    StagingRing* acquire_store_ring(detail::BatchState& b, size_t need, uint32_t depth);
    StagingRing load_ring_;
    std::vector<std::unique_ptr<StagingRing>> store_rings_;
    size_t staging_peak_ = 0;
    CopyRunStats copy_stats_;  // guarded by io_mu_
    std::mutex io_mu_;  // one batch enqueues at a time

    mutable std::mutex mu_;
    std::unordered_map<QueryId, QueryState> queries_;
};

}  // namespace tkv
