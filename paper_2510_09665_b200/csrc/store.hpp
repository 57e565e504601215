// The pinned host tier (mirror of TieredStore's RAM tier,
// include/tierkv/store.hpp:142-262, src/store.cpp).
//
// Same slot geometry as the reference RAM slab (store.cpp:96-102): a
// pre-allocated slab of fixed slots of L * chunk_size * bpt bytes, one chunk
// per slot, payload layer-major [L][T][bpt] with layer l at offset l*T*bpt
// (store.cpp:343-345, 703-709). The slab is cudaHostAlloc'ed
// (Mapped|Portable), so the gather kernel writes a chunk straight into its
// slot over PCIe and the copy engine reads slot slices for loads.
//
// Same index semantics: digest-keyed entries, `writing` -> `present` only
// after the bytes landed (store.cpp:333-357), idempotent duplicate puts
// (:322-329), geometry checks (:439-443, 454-470), LRU eviction of present,
// unpinned, unshared entries (:198-263), share counts that block eviction
// and clear while a transfer reads a slot (:687-701, 836), pin and clear
// (:808-862). Disk / remote tiers, codecs and the event pump are out of
// scope.
#pragma once

#include <condition_variable>
#include <memory>
#include <mutex>
#include <optional>
#include <unordered_map>
#include <vector>

#include "common.hpp"

namespace tkv {

struct StoreConfig {
    ModelSpec model;
    size_t chunk_size = 256;
    size_t ram_pool_bytes = 64ull << 20;
};

struct StoreStats {
    size_t entries = 0;
    size_t ram_slots_total = 0;
    size_t ram_slots_used = 0;
    size_t ram_entries = 0;
};

struct ClearResult {
    size_t removed = 0;
    size_t refused = 0;
};

namespace detail {
struct PutState {
    std::mutex m;
    std::condition_variable cv;
    bool done = false;
    Status status;
};
}  // namespace detail

// Awaitable completion of one chunk write (store.hpp:58-76).
class PutHandle {
public:
    PutHandle() = default;
    explicit PutHandle(std::shared_ptr<detail::PutState> st) : st_(std::move(st)) {}
    const Status& wait() const;
    bool done() const;
    static PutHandle immediate(Status st);

private:
    std::shared_ptr<detail::PutState> st_;
};

// A reserved slot about to be written by the device.
struct SlotWrite {
    // none: no slot claimed (reservation failed, or not attempted).
    // dropped: the reference would write this chunk and evict it again before
    // its batch ends (a later put of the same batch takes the slot); it is
    // reported stored and no bytes move (begin_write_batch).
    enum class Kind { none, write, already_present, in_flight, dropped } kind = Kind::none;
    uint8_t* host = nullptr;   // slot base (host address)
    uint8_t* dev = nullptr;    // slot base (device-visible alias)
    PutHandle handle;          // completes when the bytes are present
};

// A slot pinned against eviction/clear while a transfer reads it.
struct SlotRead {
    uint8_t* host = nullptr;
    uint8_t* dev = nullptr;
    uint32_t token_count = 0;
};

class TieredStore {
public:
    explicit TieredStore(StoreConfig cfg);
    ~TieredStore();
    TieredStore(const TieredStore&) = delete;
    TieredStore& operator=(const TieredStore&) = delete;

    const StoreConfig& config() const { return cfg_; }
    size_t slot_bytes() const { return slot_bytes_; }
    size_t slab_slots() const { return slot_bytes_ ? slab_.bytes / slot_bytes_ : 0; }

    // --- device write path (used by the connector's K1 store) --------------
    // Claims a slot for `digest` (token_count rows per layer). Errors:
    // invalid_argument for geometry mismatch, tier_full when no slot can be
    // freed. The entry stays invisible to contains() until commit_write.
    Result<SlotWrite> begin_write(const Digest& digest, uint32_t token_count, bool pin);
    // The slots of one store batch, claimed up front with the outcome of the
    // reference's sequential batch_put (store.cpp:332-357, 500-506): puts are
    // applied in order, and a put that finds no free slot evicts the least
    // recently touched entry that is present, unpinned and unshared — where
    // chunks this same batch is loading count as unshared (their loads finish
    // before the reference seals the batch) and the batch's own earlier
    // writes count as present (the reference has written them by then; such a
    // victim comes back as Kind::dropped). `own_shares`: digest -> shares this
    // batch holds through acquire(). One deliberate difference: a chunk this
    // batch loads is only evictable by a put of at most its token count (the
    // new bytes land behind the loads layer by layer); the reference, which
    // seals after the loads, could also pick it for a longer chunk.
    struct WriteSpec {
        Digest digest;
        uint32_t token_count = 0;
        bool pin = false;
    };
    // `touch_order` receives the digests in the order the reference's writes
    // touch them (new writes, repeated puts, already-present puts); replay it
    // with commit_batch() once the batch's bytes landed.
    std::vector<Result<SlotWrite>> begin_write_batch(
        const std::vector<WriteSpec>& specs,
        const std::unordered_map<Digest, uint32_t, DigestHasher>& own_shares,
        std::vector<Digest>* touch_order = nullptr);
    // A whole store batch landed: every written entry becomes present, the
    // touch order is replayed, and only then are the put handles finished.
    // Safe to call from a CUDA host callback.
    void commit_batch(const std::vector<Digest>& digests, const std::vector<Digest>& touches);
    // Marks the entry present (ok) or drops the claim (error). Safe to call
    // from a CUDA host callback (no CUDA API calls inside).
    void commit_write(const Digest& digest, const Status& status);

    // --- device read path (used by the connector's K2 load) ----------------
    // Shares the entry (blocks eviction/clear) if present with the expected
    // token count; release() when the transfer finished.
    Result<SlotRead> acquire(const Digest& digest, uint32_t expect_tokens);
    void release(const Digest& digest);

    // --- reference-shaped API (store.hpp:153-171) ---------------------------
    // Host payload put ([L][T][bpt]), synchronous; used to seed the tier.
    PutHandle put(const Digest& digest, uint32_t token_count, const uint8_t* payload,
                  size_t payload_bytes, bool pin = false);
    Result<std::vector<uint8_t>> get(const Digest& digest);
    Result<std::vector<uint8_t>> get_layer(const Digest& digest, uint32_t layer);
    bool contains(const Digest& digest) const;
    // Leading entries of `digests` that are present, under one lock (the
    // reference probes contains() once per chunk, store.cpp:797-806).
    size_t present_prefix(const std::vector<Digest>& digests) const;
    // present[i] = contains(digests[i]) for every digest, under one lock.
    std::vector<bool> present_mask(const std::vector<Digest>& digests) const;
    Status pin(const Digest& digest, bool on);
    ClearResult clear(const std::vector<Digest>& digests);
    size_t evict_until(size_t bytes_needed);
    StoreStats stats() const;
    // Change feed of the present set (contains()) for a device mirror (the
    // lookup kernels' presence index, KeyHasher::enable_presence). Every
    // transition to or from `present` is recorded per subscriber, coalesced
    // to the final state per digest; drain hands them over. A subscriber's
    // first drain, or one with want_full, returns the whole present set
    // instead (reset = true: the mirror must be cleared first).
    size_t presence_subscribe();
    void presence_drain(size_t id, bool want_full, std::vector<std::pair<Digest, bool>>& out, bool& reset);

    // LMCK record framing (chunk_file.cpp:7-95) for interop with the
    // reference's disk / wire format: export a present entry as a record,
    // or import a record (checksum and geometry verified) into a slot.
    Result<std::vector<uint8_t>> export_record(const Digest& digest, uint64_t model_tag_hash);
    // Into a caller buffer: *n = record bytes always; bytes written only when
    // out != nullptr and cap >= *n (a size query costs no copy or checksum).
    Status export_record_into(const Digest& digest, uint64_t model_tag_hash, uint8_t* out, size_t cap,
                              size_t* n);
    Status import_record(const uint8_t* record, size_t n, bool pin = false);

private:
    struct Entry {
        enum class State : uint8_t { writing, present };
        State state = State::writing;
        uint16_t token_count = 0;
        uint32_t slot = 0;
        bool pinned = false;
        uint32_t share_count = 0;
        uint64_t last_touch = 0;
        std::shared_ptr<detail::PutState> writer;  // set while writing
    };

    bool reserve_slot_locked(uint32_t& slot);
    size_t evict_until_locked(size_t bytes_needed);
    void touch(Entry& e) { e.last_touch = ++clock_; }

    StoreConfig cfg_;
    size_t slot_bytes_ = 0;
    PinnedBuffer slab_;
    mutable std::mutex mu_;
    std::unordered_map<Digest, Entry, DigestHasher> index_;
    std::vector<uint32_t> free_slots_;
    uint64_t clock_ = 0;
    void presence_changed(const Digest& d, bool present);  // caller holds mu_
    // Pending changes of one subscriber, one final state per digest: a
    // contiguous vector (drained by a swap) indexed by a flat open-addressing
    // table (the drain is on the lookup path; a node-based map measured ~75 ns
    // per entry to walk there).
    struct PresenceFeed {
        std::vector<std::pair<Digest, bool>> pending;
        std::vector<int32_t> index;  // power of two, -1 = empty; >= 2 x pending
        bool fresh = true;           // nothing drained yet: the first drain is a full snapshot
        void note(const Digest& d, bool present);
        void clear();
    };
    std::vector<std::unique_ptr<PresenceFeed>> feeds_;  // guarded by mu_
};

}  // namespace tkv
