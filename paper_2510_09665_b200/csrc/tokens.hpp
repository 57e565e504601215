// Chunking and chunk keys (mirror of include/tierkv/tokens.hpp:13-73).
//
// The arithmetic is the reference's: 256-token spans (only the last may be
// short), digest_i = SHA-256(u16le(|tag|) | tag | digest_{i-1} | u32le tokens).
// The difference is where it runs: every digest is computed by the K3 kernel
// (sha256_chain.cu) through a KeyHasher, one warp per sequence, and a
// sequence is hashed ONCE per query — the reference re-derives the same chain
// three to four times (connector.cpp:74,103,139,446-450).
#pragma once

#include <functional>
#include <mutex>
#include <string>
#include <unordered_set>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"

namespace tkv {

struct ChunkSpan {
    size_t start = 0;
    size_t end = 0;
    size_t length() const { return end - start; }
    bool operator==(const ChunkSpan&) const = default;
};

struct ChunkKey {
    Digest digest = kZeroDigest;
    std::string model_tag;
    uint32_t chunk_index = 0;
    bool operator==(const ChunkKey& o) const { return digest == o.digest; }  // tokens.hpp:33
};

// tokens.cpp:7-15. Throws std::invalid_argument for chunk_size < 1.
std::vector<ChunkSpan> chunk_tokens(size_t n_tokens, size_t chunk_size);

// Device SHA-256 chain engine. Thread-safe (one launch at a time).
class KeyHasher {
public:
    KeyHasher(std::string model_tag, size_t chunk_size, int device = -1);

    const std::string& model_tag() const { return tag_; }
    size_t chunk_size() const { return chunk_size_; }

    // Digests of every chunk of every sequence, in one kernel launch.
    // parents (optional, one per sequence) resume a chain (KeyChain::reset).
    std::vector<std::vector<Digest>> hash(const std::vector<TokenSpanView>& seqs,
                                          const std::vector<Digest>* parents = nullptr);
    std::vector<Digest> hash_one(TokenSpanView seq, const Digest& parent = kZeroDigest);

    // Lookup form: the leading digests of each sequence, just far enough to
    // decide its longest stored prefix — like the reference's
    // longest_prefix_match (tokens.cpp:59-69), which stops at the first
    // absent chunk. `present(d)` returns how many leading digests of d are
    // stored. Memo hits come from the parallel probe (verified); past them
    // one SHA chunk decides, and only a present one continues the chain.
    // `while_waiting` (optional) runs on the calling thread while the first
    // launch is in flight (the caller's own host work, off the critical path).
    // `present_rows` (optional) receives, per sequence, how many leading
    // chunks are stored: decided on the device from the presence index (see
    // set_presence) in the same launches — or, where the device could not
    // decide (no index, a memo hit that failed verification, a stored chunk
    // the memo had no link for), by `present` on the host.
    using PresentPrefix = std::function<size_t(const std::vector<Digest>&)>;
    // `mapped` (optional): per sequence, a mapped pinned buffer that
    // `while_waiting` fills with that sequence's tokens; when the lookup runs
    // its kernels after while_waiting, they read the tokens there (no
    // staging copy of the prompts).
    std::vector<std::vector<Digest>> hash_prefix(const std::vector<TokenSpanView>& seqs,
                                                 const PresentPrefix& present,
                                                 const std::function<void()>& while_waiting = {},
                                                 std::vector<size_t>* present_rows = nullptr,
                                                 const std::vector<const TokenId*>* mapped = nullptr);
    // A device mirror of the tier's present set (PresenceView), probed by the
    // lookup kernels (needs the memo): lookups then decide the stored prefix
    // without the host index. `drain(want_full, changes, reset)` hands over
    // the tier's pending changes (TieredStore::presence_drain); they are
    // applied by each lookup's first kernel. max_entries: the tier's slots.
    using PresenceDrain = std::function<void(bool, std::vector<std::pair<Digest, bool>>&, bool&)>;
    void enable_presence(size_t max_entries, PresenceDrain drain);
    // Lookups whose stored prefix the host decided (diagnostics / tests).
    uint64_t host_decided() const { return host_decided_; }

    // Launch counters (tests assert the once-per-query property).
    uint64_t launches() const { return launches_; }
    uint64_t chunks_hashed() const { return chunks_; }

    // Prefix-digest memo: `entries` chunk links
    // kept on the device; 0 disables. Exact: hits are verified token by token.
    void enable_memo(size_t entries);
    struct MemoStats {
        uint64_t hits = 0, misses = 0, capacity = 0, resets = 0, rehashes = 0;
        uint64_t witnessed = 0;  // lookup rows decided absent by the witness (no SHA)
    };
    MemoStats memo_stats();
    // Test hook: corrupt every memo slot's digest (hits must then fail
    // verification and be re-hashed).
    void debug_poison_memo();

private:
    void memo_reset_locked();
    MemoView stage_locked(const std::vector<TokenSpanView>& seqs, const std::vector<Digest>* parents,
                          size_t total_tokens, size_t total_chunks, size_t max_inserts, HashParams& p,
                          const std::vector<const TokenId*>* mapped = nullptr);
    void rehash_bad_locked(size_t n_chains, size_t total_chunks, const HashParams& p);
    std::string tag_;
    size_t chunk_size_;
    int device_;
    std::mutex mu_;
    Stream stream_;
    PinnedBuffer h_tokens_, h_chains_, h_out_, h_bad_, h_first_;  // mapped host side of a launch
    PinnedBuffer h_present_, h_known_;                           // lookup results per chain (mapped)
    uint64_t host_decided_ = 0;
    // presence index (device table) and the pending changes of one lookup
    void presence_sync_locked(MemoView& m);
    bool first_row_lookup(const std::vector<TokenSpanView>& seqs, const std::vector<size_t>& rows,
                          std::vector<std::vector<Digest>>& out, std::vector<size_t>& present_rows,
                          const std::function<void()>& while_waiting, bool& waited);
    PinnedBuffer h_row0_tok_, h_row0_ch_, h_row0_out_;  // first-row fast path (mapped)
    PinnedBuffer h_srcs_;                               // per-chain token sources (mapped prompts)
    std::unordered_set<uint64_t> seen_row0_;            // route hint: first chunks looked up before
    PresenceDrain presence_drain_;
    DeviceBuffer presence_table_;
    DeviceBuffer witness_table_, witness_meta_;  // absence witness W + unknown count (kernels.hpp)
    DeviceBuffer link_table_;                    // memo link index: digest -> prefix key
    PinnedBuffer h_updates_;
    uint32_t presence_mask_ = 0;
    size_t presence_used_ = 0;  // slots claimed since the table was cleared (upper bound)
    std::vector<std::pair<Digest, bool>> presence_pending_;
    DeviceBuffer d_tokens_, d_chains_, d_out_, d_hit_;  // HBM copies the kernels work on
    DeviceBuffer d_keys_, d_first_;                     // memo probe keys / first miss per chain
    uint64_t memo_rehashes_ = 0;
    uint64_t launches_ = 0, chunks_ = 0;
    // memo (device): slots, entries, counter + stats
    DeviceBuffer memo_slots_, memo_entries_, memo_meta_;
    MemoView memo_;
    size_t memo_used_bound_ = 0;  // host upper bound of inserted entries
    uint64_t memo_resets_ = 0;
};

// tokens.cpp:49-57.
std::vector<ChunkKey> chunk_keys(KeyHasher& hasher, TokenSpanView tokens);

// Incremental chain (tokens.hpp:41-63); each next() is one device launch.
class KeyChain {
public:
    explicit KeyChain(KeyHasher& hasher) : hasher_(&hasher) {}
    ChunkKey next(TokenSpanView chunk_tokens);
    const Digest& parent() const { return parent_; }
    uint32_t next_index() const { return index_; }
    void reset(const Digest& parent, uint32_t next_index) {
        parent_ = parent;
        index_ = next_index;
    }

private:
    KeyHasher* hasher_;
    Digest parent_ = kZeroDigest;
    uint32_t index_ = 0;
};

using KeyIndex = std::function<bool(const ChunkKey&)>;

// tokens.cpp:59-69 over precomputed keys: k full chunks matched -> k * cs,
// plus the partial tail when that is present too; stops at the first miss.
size_t longest_prefix_match(const std::vector<ChunkKey>& keys, size_t n_tokens, size_t chunk_size,
                            const KeyIndex& index);
size_t longest_prefix_match(KeyHasher& hasher, TokenSpanView tokens, const KeyIndex& index);

}  // namespace tkv
