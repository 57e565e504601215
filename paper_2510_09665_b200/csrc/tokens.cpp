#include "tokens.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

namespace tkv {

std::vector<ChunkSpan> chunk_tokens(size_t n, size_t chunk_size) {
    if (chunk_size < 1) throw std::invalid_argument("chunk_size must be >= 1");
    std::vector<ChunkSpan> spans;
    spans.reserve((n + chunk_size - 1) / chunk_size);
    for (size_t start = 0; start < n; start += chunk_size)
        spans.push_back({start, std::min(start + chunk_size, n)});
    return spans;
}

KeyHasher::KeyHasher(std::string model_tag, size_t chunk_size, int device)
    : tag_(std::move(model_tag)), chunk_size_(chunk_size), device_(device) {
    if (chunk_size_ < 1) throw std::invalid_argument("chunk_size must be >= 1");
    if (tag_.size() > size_t(kMaxTagBytes))
        throw std::invalid_argument("model tag longer than the device hash supports");
    if (device_ < 0) TKV_CUDA(cudaGetDevice(&device_));
    stream_ = Stream::create();
}

namespace {
// TKV_TRACE_LOOKUP=1: host-side phase times of every hash() call on stderr.
bool trace_lookup() {
    static const bool on = std::getenv("TKV_TRACE_LOOKUP") != nullptr;
    return on;
}
double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

std::vector<std::vector<Digest>> KeyHasher::hash(const std::vector<TokenSpanView>& seqs,
                                                 const std::vector<Digest>* parents) {
    const double t_in = trace_lookup() ? now_us() : 0;
    std::lock_guard lock(mu_);
    TKV_CUDA(cudaSetDevice(device_));
    size_t total_tokens = 0, total_chunks = 0;
    for (const auto& s : seqs) {
        total_tokens += s.size();
        total_chunks += (s.size() + chunk_size_ - 1) / chunk_size_;
    }
    std::vector<std::vector<Digest>> out(seqs.size());
    if (total_chunks == 0) return out;

    // Tokens, chain descriptors and digests live in mapped pinned memory: K3
    // reads and writes them over PCIe directly (a few KiB per chain), so a
    // lookup never queues on the copy engines behind in-flight KV transfers.
    h_tokens_.reserve(total_tokens * sizeof(TokenId) + 64);
    h_chains_.reserve(seqs.size() * sizeof(ChainDesc));
    h_out_.reserve(total_chunks * 32);

    auto* tok = reinterpret_cast<TokenId*>(h_tokens_.host);
    auto* ch = reinterpret_cast<ChainDesc*>(h_chains_.host);
    size_t toff = 0, row = 0;
    for (size_t i = 0; i < seqs.size(); ++i) {
        std::copy(seqs[i].begin(), seqs[i].end(), tok + toff);
        ChainDesc d;
        d.token_off = toff;
        d.n_tokens = uint32_t(seqs[i].size());
        d.out_first = uint32_t(row);
        if (parents) std::copy((*parents)[i].begin(), (*parents)[i].end(), d.parent);
        ch[i] = d;
        toff += seqs[i].size();
        row += (seqs[i].size() + chunk_size_ - 1) / chunk_size_;
    }
    HashParams p;
    p.chunk_size = uint32_t(chunk_size_);
    p.tag_len = uint32_t(tag_.size());
    std::copy(tag_.begin(), tag_.end(), p.tag);

    // Stage tokens and descriptors into HBM (one parallel read of the mapped
    // buffers), run the chains writing digests to HBM, then verify memo hits
    // and publish every digest to the mapped result buffer.
    const double t_packed = trace_lookup() ? now_us() : 0;
    const size_t tok_bytes = total_tokens * sizeof(TokenId);
    const size_t ch_bytes = seqs.size() * sizeof(ChainDesc);
    d_tokens_.reserve(tok_bytes + 64);
    d_chains_.reserve(ch_bytes + 64);
    d_out_.reserve(total_chunks * 32);
    h_bad_.reserve(seqs.size() * sizeof(unsigned int));
    auto* bad = reinterpret_cast<unsigned int*>(h_bad_.host);
    std::fill(bad, bad + seqs.size(), ~0u);
    MemoView m = memo_;
    if (memo_.slots) {
        if (memo_used_bound_ + total_chunks > memo_.entry_cap) memo_reset_locked();
        memo_used_bound_ += total_chunks;
        d_hit_.reserve(total_chunks * sizeof(uint32_t));
        d_keys_.reserve(total_chunks * sizeof(unsigned long long));
        d_first_.reserve(seqs.size() * sizeof(uint32_t));
        m = memo_;
        m.hit_entry = reinterpret_cast<uint32_t*>(d_hit_.ptr);
        m.keys = reinterpret_cast<unsigned long long*>(d_keys_.ptr);
        m.first_miss = reinterpret_cast<uint32_t*>(d_first_.ptr);
    }
    const auto* d_tok = reinterpret_cast<const uint32_t*>(d_tokens_.ptr);
    const auto* d_ch = reinterpret_cast<const ChainDesc*>(d_chains_.ptr);
    TKV_CUDA(launch_sm_copy(h_chains_.dev, d_chains_.ptr, ch_bytes, stream_));
    if (memo_.slots)  // staging + per-row fingerprints in one pass
        TKV_CUDA(launch_memo_stage(reinterpret_cast<const uint32_t*>(h_tokens_.dev),
                                   reinterpret_cast<uint32_t*>(d_tokens_.ptr), d_ch, uint32_t(seqs.size()),
                                   uint32_t(total_chunks), p, m, stream_));
    else
        TKV_CUDA(launch_sm_copy(h_tokens_.dev, d_tokens_.ptr, tok_bytes, stream_));
    TKV_CUDA(launch_hash_chains(d_tok, d_ch, uint32_t(seqs.size()), p, d_out_.ptr, stream_,
                                memo_.slots ? &m : nullptr));
    TKV_CUDA(launch_memo_verify(d_tok, d_ch, uint32_t(seqs.size()), uint32_t(total_chunks), p,
                                d_out_.ptr, memo_.slots ? &m : nullptr, h_out_.dev,
                                reinterpret_cast<unsigned int*>(h_bad_.dev), stream_));
    const double t_launched = trace_lookup() ? now_us() : 0;
    TKV_CUDA(cudaStreamSynchronize(stream_));
    const double t_synced = trace_lookup() ? now_us() : 0;
    ++launches_;
    chunks_ += total_chunks;

    // A memo hit that failed verification (a 40-bit tag collision): re-hash
    // those chains from the first bad chunk with plain SHA-256.
    std::vector<ChainDesc> redo;
    for (size_t i = 0; i < seqs.size(); ++i) {
        if (bad[i] == ~0u) continue;
        ChainDesc d = ch[i];
        const size_t skip = size_t(bad[i]) * chunk_size_;
        d.token_off += skip;
        d.n_tokens -= uint32_t(skip);
        d.out_first += bad[i];
        if (bad[i]) std::copy(h_out_.host + 32 * (d.out_first - 1), h_out_.host + 32 * d.out_first, d.parent);
        redo.push_back(d);
    }
    if (!redo.empty()) {
        ++memo_rehashes_;
        std::copy(redo.begin(), redo.end(), ch);
        TKV_CUDA(launch_sm_copy(h_chains_.dev, d_chains_.ptr, redo.size() * sizeof(ChainDesc), stream_));
        TKV_CUDA(launch_hash_chains(d_tok, d_ch, uint32_t(redo.size()), p, d_out_.ptr, stream_, nullptr));
        TKV_CUDA(launch_memo_verify(d_tok, d_ch, uint32_t(redo.size()), uint32_t(total_chunks), p,
                                    d_out_.ptr, nullptr, h_out_.dev, nullptr, stream_));
        TKV_CUDA(cudaStreamSynchronize(stream_));
    }

    row = 0;
    for (size_t i = 0; i < seqs.size(); ++i) {
        size_t n = (seqs[i].size() + chunk_size_ - 1) / chunk_size_;
        out[i].resize(n);
        for (size_t c = 0; c < n; ++c, ++row)
            std::copy(h_out_.host + 32 * row, h_out_.host + 32 * row + 32, out[i][c].begin());
    }
    if (trace_lookup())
        std::fprintf(stderr, "[tkv hash] chains=%zu rows=%zu pack=%.1fus launch=%.1fus device+sync=%.1fus unpack=%.1fus\n",
                     seqs.size(), total_chunks, t_packed - t_in, t_launched - t_packed, t_synced - t_launched,
                     now_us() - t_synced);
    return out;
}

void KeyHasher::enable_memo(size_t entries) {
    std::lock_guard lock(mu_);
    TKV_CUDA(cudaSetDevice(device_));
    if (entries == 0 || chunk_size_ > 256) {  // the memo lives in the warp-cooperative kernel
        memo_ = MemoView{};
        return;
    }
    entries = std::min<size_t>(entries, size_t(1) << 24);
    size_t slots = 1;
    while (slots < 2 * entries) slots <<= 1;
    const uint32_t words = uint32_t(17 + chunk_size_);
    memo_slots_.reserve(slots * 8 * sizeof(unsigned long long));  // 64-byte slots
    memo_entries_.reserve(entries * words * sizeof(uint32_t));
    memo_meta_.reserve(64);
    memo_.slots = reinterpret_cast<unsigned long long*>(memo_slots_.ptr);
    memo_.entries = reinterpret_cast<uint32_t*>(memo_entries_.ptr);
    memo_.counter = reinterpret_cast<unsigned int*>(memo_meta_.ptr);
    memo_.stats = reinterpret_cast<unsigned long long*>(memo_meta_.ptr + 16);
    memo_.slot_mask = uint32_t(slots - 1);
    memo_.entry_cap = uint32_t(entries);
    memo_.entry_words = words;
    TKV_CUDA(cudaMemsetAsync(memo_meta_.ptr, 0, 64, stream_));
    memo_reset_locked();
    // Keep the slot table (64 B per slot) resident in L2 for this stream's
    // kernels: a memo hit is one dependent load per chunk on the serial
    // chain, and the KV transfers between lookups (streaming loads/stores)
    // would otherwise evict it to DRAM. Best effort: ignored if unsupported.
    const size_t slot_bytes = slots * 64;
    int max_persist = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device_);
    if (max_persist > 0) {
        size_t cur = 0;
        cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
        const size_t want = std::min<size_t>(size_t(max_persist), std::max(cur, slot_bytes));
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) {
            cudaStreamAttrValue attr{};
            attr.accessPolicyWindow.base_ptr = memo_slots_.ptr;
            attr.accessPolicyWindow.num_bytes = std::min(slot_bytes, want);
            attr.accessPolicyWindow.hitRatio = 1.0f;
            attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cudaStreamSetAttribute(stream_, cudaStreamAttributeAccessPolicyWindow, &attr);
        }
        cudaGetLastError();
    }
    TKV_CUDA(cudaStreamSynchronize(stream_));
}

void KeyHasher::memo_reset_locked() {
    TKV_CUDA(cudaMemsetAsync(memo_.slots, 0, (size_t(memo_.slot_mask) + 1) * 64, stream_));
    TKV_CUDA(cudaMemsetAsync(memo_.counter, 0, sizeof(unsigned int), stream_));
    memo_used_bound_ = 0;
    ++memo_resets_;
}

KeyHasher::MemoStats KeyHasher::memo_stats() {
    std::lock_guard lock(mu_);
    MemoStats s;
    if (!memo_.slots) return s;
    unsigned long long st[2] = {0, 0};
    TKV_CUDA(cudaMemcpyAsync(st, memo_.stats, sizeof st, cudaMemcpyDeviceToHost, stream_));
    TKV_CUDA(cudaStreamSynchronize(stream_));
    s.hits = st[0];
    s.misses = st[1];
    s.capacity = memo_.entry_cap;
    s.resets = memo_resets_ - 1;  // the enabling clear is not a reset
    s.rehashes = memo_rehashes_;
    return s;
}

void KeyHasher::debug_poison_memo() {
    std::lock_guard lock(mu_);
    TKV_CUDA(launch_memo_poison(memo_, stream_));
    TKV_CUDA(cudaStreamSynchronize(stream_));
}

std::vector<Digest> KeyHasher::hash_one(TokenSpanView seq, const Digest& parent) {
    std::vector<Digest> parents{parent};
    return std::move(hash({seq}, &parents)[0]);
}

std::vector<ChunkKey> chunk_keys(KeyHasher& hasher, TokenSpanView tokens) {
    auto digests = hasher.hash_one(tokens);
    std::vector<ChunkKey> keys(digests.size());
    for (size_t i = 0; i < digests.size(); ++i)
        keys[i] = ChunkKey{digests[i], hasher.model_tag(), uint32_t(i)};
    return keys;
}

ChunkKey KeyChain::next(TokenSpanView tokens) {
    if (tokens.empty() || tokens.size() > hasher_->chunk_size())
        throw std::invalid_argument("chunk token count out of range");  // tokens.cpp:23-24
    auto d = hasher_->hash_one(tokens, parent_);
    ChunkKey key{d.at(0), hasher_->model_tag(), index_};
    parent_ = key.digest;
    ++index_;
    return key;
}

size_t longest_prefix_match(const std::vector<ChunkKey>& keys, size_t n_tokens, size_t chunk_size,
                            const KeyIndex& index) {
    size_t matched = 0;
    for (size_t i = 0; i < keys.size(); ++i) {
        if (!index(keys[i])) break;
        matched = std::min(n_tokens, (i + 1) * chunk_size);
    }
    return matched;
}

size_t longest_prefix_match(KeyHasher& hasher, TokenSpanView tokens, const KeyIndex& index) {
    return longest_prefix_match(chunk_keys(hasher, tokens), tokens.size(), hasher.chunk_size(),
                                index);
}

}  // namespace tkv
