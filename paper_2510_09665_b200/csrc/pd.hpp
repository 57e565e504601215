// Prefill -> decode disaggregation over NVLink (replaces the TCP PD_PUSH path
// of run_pd, src/sim_engine.cpp:374-472, and the decoder landing area
// PdStaging, include/tierkv/pd_staging.hpp, src/pd_staging.cpp).
//
// Data plane: the prefiller's K1 gathers each chunk's [L][T][bpt] payload
// straight out of its pages into the decoder's landing buffer — a device
// address on the decoder GPU reached over NVLink (peer access in one process,
// a CUDA IPC mapping across processes). No host bytes, no record encode, no
// FNV. The decoder then scatters every landed chunk into its own pages with
// ONE K2 launch over all chunks and layers.
//
// Control plane: PdStaging keeps the reference's contract unchanged —
// register before any push; each ordinal is filled exactly once (a duplicate
// push acks without overwriting); a push beyond the final ordinal, or a final
// marker below an already filled ordinal, is a protocol_error; await returns
// the records in ordinal order once the final ordinal and everything before
// it landed, then forgets the query; cancel wakes the awaiter with io_error.
// A record here describes where the payload landed instead of carrying it.
#pragma once

#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"
#include "paged_store.hpp"

namespace tkv {

struct DevicePlan;  // copy_plan.hpp

struct PdRecord {
    uint64_t addr = 0;          // device address of the landed chunk payload (decoder GPU)
    uint64_t bytes = 0;
    uint32_t token_count = 0;
    uint32_t first_token = 0;   // absolute position of the chunk's first token
};

class PdStaging {
public:
    Status register_query(QueryId id);
    Status push(QueryId id, uint32_t ordinal, bool last, const PdRecord& rec);
    // Blocks until complete (or cancelled); records in ordinal order.
    Result<std::vector<PdRecord>> await(QueryId id);
    Status cancel(QueryId id);
    size_t registered() const;

private:
    // One landing per registered query. Records arrive out of order (one per
    // chunk, or per layer-window of a layer-streamed send) and are kept
    // unsorted; the landing is complete when the final ordinal is known and
    // every ordinal up to it is filled (ordinals past it are refused, so a
    // count suffices). Each awaiter sleeps on its own query's condition.
    struct Landing {
        std::unordered_map<uint32_t, PdRecord> filled;
        uint32_t highest = 0;     // largest filled ordinal (when filled is not empty)
        bool final_known = false;
        uint32_t final_ordinal = 0;
        bool cancelled = false;
        std::condition_variable wake;
        bool done() const { return final_known && filled.size() == size_t(final_ordinal) + 1; }
    };
    mutable std::mutex mu_;
    std::unordered_map<QueryId, std::shared_ptr<Landing>> landings_;
};

// Prefiller side: K1 over chunks [first_chunk, first_chunk + n_chunks) of the
// query's first n_tokens tokens, all layers, into `landing` laid out as
// consecutive chunk payloads (chunk i at landing + i * chunk_stride bytes,
// each [L][T_i][bpt]). `landing` may be a peer GPU's memory. Enqueued on
// `stream`; returns the records describing where each chunk landed.
Result<std::vector<PdRecord>> pd_send_chunks(PagedKVStore& pages, QueryId query, size_t n_tokens,
                                             size_t chunk_size, uint64_t landing,
                                             uint64_t chunk_stride, cudaStream_t stream,
                                             int ctas = 0);

// Same contract through the copy engines: K1 gathers groups of chunks into
// `staging` (local HBM, same layout as landing) on `stream` while the copy
// engine moves each finished group to `landing` with one peer memcpy on a
// second stream (groups of about `group_bytes`). One extra HBM pass; the
// NVLink leg is a plain CE peer copy (the measured 770 GB/s path).
Result<std::vector<PdRecord>> pd_send_chunks_staged(PagedKVStore& pages, QueryId query, size_t n_tokens,
                                                    size_t chunk_size, uint64_t landing,
                                                    uint64_t chunk_stride, uint64_t staging,
                                                    cudaStream_t stream, uint64_t group_bytes = 1ull << 30);

// Layer-streamed send at chunk or page granularity (run_pd's PdGranularity,
// src/sim_engine.cpp:389-424: unit_tokens = chunk_size or page_tokens; one
// record per unit, [L][T_unit][bpt] at landing + i * unit_stride). The K1 plan
// is built once; send_layer(l) gathers layer l of every unit straight into
// the landing buffer on the sender's own stream, ordered after an event on
// the engine stream, so the NVLink transfer of layer l overlaps the prefill
// compute of the layers after it (the reference ships only after the whole
// prefill). finish() waits for the last layer and returns the records, which
// the caller then pushes (ordinals per unit) to the decoder's PdStaging.
class PdLayerSender {
public:
    PdLayerSender(PagedKVStore& pages, QueryId query, size_t n_tokens, size_t unit_tokens, uint64_t landing,
                  uint64_t unit_stride);
    ~PdLayerSender();
    PdLayerSender(const PdLayerSender&) = delete;
    PdLayerSender& operator=(const PdLayerSender&) = delete;
    const Status& status() const { return status_; }  // construction outcome
    Status send_layer(uint32_t layer, cudaStream_t engine_stream);
    Result<std::vector<PdRecord>> finish();

private:
    PagedKVStore& pages_;
    QueryId query_;
    size_t n_tokens_, unit_tokens_;
    Status status_;
    std::vector<PdRecord> recs_;
    std::unique_ptr<DevicePlan> plan_;
    Stream stream_;
    std::vector<bool> sent_;
};

// Decoder side: K2 of every landed record into the query's pages (all
// layers, one launch), marks the pages populated. Enqueued on `stream`.
Status pd_land_chunks(PagedKVStore& pages, QueryId query, const std::vector<PdRecord>& records,
                      cudaStream_t stream, int ctas = 0);

// Peer access between two devices of this process (idempotent).
Status enable_peer_access(int device, int peer);

}  // namespace tkv
