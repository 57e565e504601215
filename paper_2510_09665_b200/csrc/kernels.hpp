// Launch interface of the sm_100a kernels. POD structs only: these are what
// the host C++ (and the C-ABI in include/tierkv_b200.h) hand to the device.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tkv {

// Count of kernel launches issued by this library (bench.py's gpu_launches).
void note_launch();
uint64_t launch_count();

// ---------------------------------------------------------------------------
// K1/K2: multi-layer paged KV gather (store) and scatter (retrieve).
//
// Replaces PagedKVStore::gather_tokens_into / scatter_tokens
// (src/paged_store.cpp:123-175) as called per (layer, chunk) from
// Connector::start_store_kv (src/connector.cpp:300-323) and
// Connector::run_load_layer (src/connector.cpp:179-219): ONE launch moves
// every chunk descriptor of a batch for a range of layers.
//
// Paged side. Reference layout (paged_store.hpp:19-82): a page holds
// page_tokens rows of ONE layer, row = bpt opaque bytes, page p at
// base + p * page_stride; each (query, layer) has its own page list.
// vLLM layout: per-layer tensors [planes=2 (K,V)][blocks][page_tokens][H*D],
// one block table shared by all layers; the chunk row is K(H*D) | V(H*D).
// Both are expressed by PagedLayout.
struct PagedLayout {
    uint64_t base = 0;                // pool base (used when layer_base == nullptr)
    const uint64_t* layer_base = nullptr;  // optional device array [num_layers]
    uint64_t page_stride = 0;         // bytes between consecutive page ids
    uint64_t plane_stride = 0;        // bytes between the K and V planes
    uint32_t token_stride = 0;        // bytes between rows inside a page
    uint32_t plane_bytes = 0;         // bytes of one row in one plane
    uint32_t n_planes = 1;            // 1 = opaque row, 2 = K|V planes
    uint32_t page_tokens = 16;
    uint32_t bpt = 0;                 // chunk row bytes = n_planes * plane_bytes
    uint32_t shared_table = 0;        // 1: page-table row 0 serves every layer
};

// One chunk transfer (a ChunkDescriptor of a load or store plan,
// connector.hpp:22-43). Spans start on a chunk boundary, hence page-aligned
// (ModelSpec::validate requires page_tokens | chunk_size).
struct XferDesc {
    uint64_t chunk = 0;          // device-visible chunk base: HBM, mapped pinned host, or peer
    uint64_t layer_stride = 0;   // bytes between layers in the chunk buffer (slot: T*bpt)
    const int32_t* table = nullptr;  // device page table, [layers][table_stride]
    uint32_t table_stride = 0;
    uint32_t first_page = 0;     // span.start / page_tokens
    uint32_t n_tokens = 0;       // rows to move (span length; may clip a record)
    uint32_t pad = 0;
};

enum class CopyDir : int { gather = 0, scatter = 1 };  // gather: pages -> chunk

struct PagedCopyPlan {
    const XferDesc* descs = nullptr;   // device
    const uint32_t* tile_base = nullptr;  // device, [n_desc + 1] prefix of tiles
    uint32_t n_desc = 0;
    uint32_t total_tiles = 0;
    uint32_t layer_begin = 0;
    uint32_t n_layers = 1;             // layers moved by this launch
    uint32_t pages_per_tile = 1;
    uint64_t addr_or = 0;              // OR of every desc chunk base and layer stride (alignment)
    // Affine one-layer plan (0 pages = not affine): descriptor i moves
    // aff_pages pages from page-table column aff_first_page + i * aff_pages of
    // aff_table into aff_chunk0 + i * aff_chunk_stride, every descriptor full
    // but the last (aff_last_tokens rows). The unit kernel then computes every
    // address from these fields: the page id is its only dependent load.
    uint32_t aff_pages = 0;
    uint32_t aff_last_tokens = 0;
    uint32_t aff_first_page = 0;
    uint32_t aff_table_stride = 0;
    const int32_t* aff_table = nullptr;
    uint64_t aff_chunk0 = 0;
    uint64_t aff_chunk_stride = 0;
    uint64_t aff_layer_stride = 0;
};

// Tiles of one descriptor for a launch over n_layers (host + device agree).
inline uint32_t tiles_for(uint32_t n_tokens, uint32_t page_tokens, uint32_t pages_per_tile,
                          uint32_t n_layers) {
    uint32_t pages = (n_tokens + page_tokens - 1) / page_tokens;
    return n_layers * ((pages + pages_per_tile - 1) / pages_per_tile);
}

// Launches the copy; `ctas` = grid size (0 = 2 x SM count). Returns launch error.
cudaError_t launch_paged_copy(const PagedLayout& layout, const PagedCopyPlan& plan, CopyDir dir,
                              int ctas, cudaStream_t stream);
// The unit kernel over an affine plan alone (aff_* set; descs / tile_base
// unused), any launch size.
cudaError_t launch_paged_copy_affine(const PagedLayout& layout, const PagedCopyPlan& plan, CopyDir dir,
                                     int ctas, cudaStream_t stream);

// ---------------------------------------------------------------------------
// K3: chained SHA-256 chunk keys (KeyChain::next, src/tokens.cpp:22-42).
// digest_i = SHA-256(u16le(|tag|) | tag | digest_{i-1} | u32le tokens of chunk i)
// One warp per chain (request); chains are independent.
struct ChainDesc {
    uint64_t token_off = 0;     // first token in the packed token buffer
    uint32_t n_tokens = 0;      // tokens of this chain (chunked by chunk_size)
    uint32_t out_first = 0;     // first digest row of this chain in `out`
    uint8_t parent[32] = {};    // KeyChain::reset parent (zeros for a fresh chain)
};

inline constexpr int kMaxTagBytes = 256;
struct HashParams {
    uint32_t chunk_size = 256;
    uint32_t tag_len = 0;
    uint8_t tag[kMaxTagBytes] = {};
};

// Presence index of the pinned tier (TieredStore "present" entries, the
// reference's contains(), store.cpp:797-806), probed by the lookup kernels:
// an HBM open-addressing table (linear probing) of 64-byte slots
// {digest bytes as 8 words, state: 0 empty, 1 present, 2 gone (tombstone),
// 3 being claimed}. The store records every transition to and from
// `present` (TieredStore::presence_drain); each lookup hands the pending
// ones (coalesced: one final state per digest) to its first kernel, which
// applies them in parallel before the probe kernel runs (stream order).
// Distinct digests never touch each other's slots except through CAS claims
// of empty slots, so the parallel apply is race-free. Home slot: the
// digest's first 4 bytes (little-endian) & mask.
//
// Absence witness (round 2): with `witness` set, the apply also keeps the set
// W of prefix keys (the memo's probe key, a fingerprint of the whole token
// prefix) of every present digest, found through the link index (digest ->
// prefix key, filled by every memo insertion). A present digest whose key is
// unknown (hashed without this memo, or before a memo reset) is counted in
// *unknown instead. While *unknown == 0, a row whose prefix key is not in W
// is absent from the tier without computing its SHA-256: equal digests mean
// equal prefixes (the assumption the digest keys rest on), and equal
// prefixes have equal keys. A key in W only means "maybe": the row is then
// hashed as before. Presence slot words 9-10 keep the key counted at the
// digest's add (word 11: 1 = in W, 2 = unknown), so its removal undoes
// exactly that.
struct PresenceView {
    uint32_t* slots = nullptr;            // device, [mask + 1] x 16 words
    uint32_t mask = 0;
    const uint32_t* updates = nullptr;    // device-visible (mapped host): n_updates x {digest words[8], present}
    uint32_t n_updates = 0;
    unsigned long long* witness = nullptr;  // [mask + 1] x {key, count}: W (optional)
    unsigned int* unknown = nullptr;        // present digests with no known key
    const uint32_t* links = nullptr;        // link index, [link_mask + 1] x 16 words
    uint32_t link_mask = 0;
};

// Lookup outputs of the memo probe / hash kernels with a presence index:
// per chain, present_out[c] = leading rows of the chain that are present
// (bit 31 set when that decides the prefix: the next row is absent or the
// chain ended), known_out[c] = rows whose digests are in `out` ([0, known)).
struct LookupOut {
    uint32_t* present_out = nullptr;  // mapped host
    uint32_t* known_out = nullptr;    // mapped host
};

// Prefix-digest memo: a device hash table from a
// fingerprint of the whole token prefix (chain parent + every token up to the
// end of chunk k) to digest_k. Because the probe key does not contain
// digest_{k-1}, every chunk of every chain is probed in parallel
// (memo_probe_kernel); a hit is then verified exactly against its entry —
// parent digest = the previous row's digest, token count and every token — so
// a verified hit is the digest the SHA chain would have produced. Chains are
// hashed with SHA from their first miss on and the new links inserted by the
// same launch. Slot word = (tag40 << 24) | entry index;
// entry = parent[8] | digest[8] | n | tokens[chunk_size] (u32 words).
struct MemoView {
    unsigned long long* slots = nullptr;  // [slot_mask + 1] x 8 u64: tagword | digest[8 x u32]
    uint32_t* hit_entry = nullptr;        // per output row: memo entry used, or ~0u
    unsigned long long* keys = nullptr;   // per output row: prefix fingerprint (probe key)
    uint32_t* first_miss = nullptr;       // per chain: first row the probes missed
    uint32_t* entries = nullptr;          // [entry_cap][entry_words]
    unsigned int* counter = nullptr;      // next free entry
    uint32_t slot_mask = 0;
    uint32_t entry_cap = 0;               // <= 2^24
    uint32_t entry_words = 0;             // 17 + chunk_size
    unsigned long long* stats = nullptr;  // [0] hits, [1] misses, [2] rows the witness decided (optional)
    uint32_t max_rows = 0;                // hash at most this many rows per chain (0 = all)
    uint32_t* first_miss_out = nullptr;   // verify also publishes first_miss here (mapped host)
    PresenceView presence;                // optional: decide the stored prefix on the device
    LookupOut lookup;                     // with presence: per-chain results (mapped host)
    uint32_t* first_absent = nullptr;     // with presence: per chain, first memo hit that is absent
    // link index: digest -> prefix key of every inserted link (64-byte slots
    // {digest bytes as 8 words, state, key lo, key hi}); feeds the witness
    uint32_t* links = nullptr;
    uint32_t link_mask = 0;
};

// With a memo whose first_miss is set: probes every row of every chain in
// parallel (one CTA per chain), then hashes each chain from its first miss.
// With first_miss unset: hashes every row of each chain, inserting the links
// under memo.keys[row]. Without a memo: plain chains.
cudaError_t launch_hash_chains(const uint32_t* tokens, const ChainDesc* chains, uint32_t n_chains,
                               const HashParams& params, uint8_t* out, cudaStream_t stream,
                               const MemoView* memo = nullptr);
// Cold-lookup fast path: row 0 of every chain decided in one launch (tokens
// and descriptors may be mapped host memory): memo hit (verified) or SHA,
// memo insert, presence probe. digests_out[8 c..8 c+8) = digest bytes,
// flags_out[c] = 1 | 2 * present, stored last with a system-scope release.
// one (optional, n_chains == 1, fresh chain): the row's tokens by value.
struct FirstRowInline {
    uint32_t n = ~0u;      // tokens in row 0 (~0u: not used)
    uint32_t tok[256] = {};
};
cudaError_t launch_first_row(const uint32_t* tokens, const ChainDesc* chains, uint32_t n_chains,
                             const HashParams& params, const MemoView& memo, uint32_t* digests_out,
                             uint32_t* flags_out, cudaStream_t stream, unsigned long long* trace = nullptr,
                             const FirstRowInline* one = nullptr);
// Applies a presence view's pending changes (before the lookup kernels).
cudaError_t launch_presence_apply(const PresenceView& view, cudaStream_t stream);
// The memo probe pass alone (fills out / hit_entry / first_miss).
cudaError_t launch_memo_probe(const ChainDesc* chains, uint32_t n_chains, const HashParams& params,
                              uint8_t* out, const MemoView& memo, cudaStream_t stream);
// SM-driven copy of exactly `bytes` between device-visible addresses (no copy
// engine): 16-byte vectors when both ends are 16-aligned, bytes otherwise.
cudaError_t launch_sm_copy(const void* src, void* dst, uint64_t bytes, cudaStream_t stream);
// Memo pass 1: stages the packed tokens (src: mapped host) into dst (HBM)
// and writes every row's chunk fingerprint to memo.keys (chains: device).
// chain_src (optional, device-visible): per chain, the address its tokens
// are read from instead of src + token_off (prompts already in mapped memory).
cudaError_t launch_memo_stage(const uint32_t* src, uint32_t* dst, const ChainDesc* chains, uint32_t n_chains,
                              uint32_t total_rows, const HashParams& params, const MemoView& memo,
                              cudaStream_t stream, const unsigned long long* chain_src = nullptr);
// Same, taking the descriptors from mapped host memory and staging them into
// chains_dev in the same launch (a separate copy only for > 128 chains).
cudaError_t launch_memo_stage_chains(const uint32_t* src, uint32_t* dst, const ChainDesc* chains_host,
                                     ChainDesc* chains_dev, uint32_t n_chains, uint32_t total_rows,
                                     const HashParams& params, const MemoView& memo, cudaStream_t stream,
                                     const unsigned long long* chain_src = nullptr);
// Verifies every memo hit of a launch against its entry and publishes all
// digest rows from dev_out to out; first_bad[chain] = first failed chunk.
cudaError_t launch_memo_verify(const uint32_t* tokens, const ChainDesc* chains, uint32_t n_chains,
                               uint32_t total_rows, const HashParams& params, const uint8_t* dev_out,
                               const MemoView* memo, uint8_t* out, unsigned int* first_bad,
                               cudaStream_t stream);
// Test hook: corrupt the digest of every published memo slot.
cudaError_t launch_memo_poison(const MemoView& memo, cudaStream_t stream);
// SHA-256 of n bytes (one thread; for the model tag hash, hash.cpp:41-44).
cudaError_t launch_sha256_bytes(const uint8_t* data, uint32_t n, uint8_t* out, cudaStream_t stream);

// ---------------------------------------------------------------------------
// q8-scale codec (src/codec.cpp:27-91) over a batch of chunk payloads.
// Encode: src = payload, dst = blob (8 + bytes/2 + bytes%2), bytes = payload
// length. Decode: src = blob, dst = payload, bytes = original length.
// seg_base = prefix over items of codec_segments(bytes) (n + 1 entries).
struct CodecItem {
    const uint8_t* src = nullptr;
    uint8_t* dst = nullptr;
    uint64_t bytes = 0;
};
uint32_t codec_segments(uint64_t bytes);
inline uint64_t q8_blob_bytes(uint64_t payload) { return 8 + payload / 2 + (payload & 1); }
// maxabs: q8_encode_scratch_bytes(n_items) of per-call scratch (absmax per
// item, then the single-pass encode's arrival and done counters per item)
uint64_t q8_encode_scratch_bytes(uint32_t n);
cudaError_t launch_q8_encode(const CodecItem* items, const uint32_t* seg_base, uint32_t n_items,
                             uint32_t total_segs, int* maxabs, cudaStream_t stream);
cudaError_t launch_q8_decode(const CodecItem* items, const uint32_t* seg_base, uint32_t n_items,
                             uint32_t total_segs, cudaStream_t stream);

// ---------------------------------------------------------------------------
// K4: synthetic KV (synth_token_kv, src/synth.cpp:7-20) written straight into
// pages for tokens [pos_begin, pos_end) of one query over layers
// [layer_begin, layer_end). Word at byte offset i of a row is
// splitmix64(base + i), base = splitmix64(seed ^ tok<<32 ^ layer<<16 ^ splitmix64(pos)).
struct SynthArgs {
    const uint32_t* tokens = nullptr;  // device, the query's prompt (absolute positions)
    const int32_t* table = nullptr;    // device page table [layers][table_stride]
    uint32_t table_stride = 0;
    uint64_t seed = 0;
    uint32_t pos_begin = 0, pos_end = 0;
    uint32_t layer_begin = 0, layer_end = 0;
    uint64_t row_offset = 0;  // byte offset of this row slice in the full row (TP head shard)
};
cudaError_t launch_synth_pages(const PagedLayout& layout, const SynthArgs& args,
                               cudaStream_t stream);
// Counts rows (layer, token) whose page bytes differ from synth; adds to *mismatches.
cudaError_t launch_verify_pages(const PagedLayout& layout, const SynthArgs& args,
                                unsigned long long* mismatches, cudaStream_t stream);
// Adds to *mismatches the 8-byte words of a chunk payload [n_layers][n][bpt]
// (any device-visible address: HBM or a mapped pinned tier slot) that differ
// from synth for tokens [start, start + n), row slice at row_offset.
cudaError_t launch_verify_chunk(const uint32_t* tokens, uint64_t seed, uint32_t start, uint32_t n,
                                uint32_t n_layers, uint32_t bpt, uint64_t row_offset, const uint8_t* chunk,
                                unsigned long long* mismatches, cudaStream_t stream);
// Synthetic chunk payload [n_layers][n][bpt] into a flat device buffer.
cudaError_t launch_synth_chunk(const uint32_t* tokens, uint64_t seed, uint32_t start, uint32_t n,
                               uint32_t n_layers, uint32_t bpt, uint8_t* out,
                               cudaStream_t stream);

}  // namespace tkv
