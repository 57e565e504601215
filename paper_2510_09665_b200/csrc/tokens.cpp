#include "tokens.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "host_copy.hpp"

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
// Size for a per-call buffer: the next power of two (64 KiB at least), so
// prompts of varying length do not regrow it — a regrowth calls cudaMalloc /
// cudaHostAlloc, which wait for the device (behind whatever KV transfers are
// in flight: a 120 ms stall was traced in config 4 before this).
size_t grow(size_t n) {
    size_t p = size_t(64) << 10;
    while (p < n) p <<= 1;
    return p;
}

// TKV_TRACE_LOOKUP=1: host-side phase times of every hash() call on stderr.
bool trace_lookup() {
    static const bool on = std::getenv("TKV_TRACE_LOOKUP") != nullptr;
    return on;
}
double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

// Packs the sequences into the mapped buffers and stages them into HBM on the
// hasher stream (with the memo: the fingerprint pass does the staging).
// Caller holds mu_. Returns the memo view for this launch (slots == nullptr
// without a memo).
MemoView KeyHasher::stage_locked(const std::vector<TokenSpanView>& seqs, const std::vector<Digest>* parents,
                                 size_t total_tokens, size_t total_chunks, size_t max_inserts, HashParams& p,
                                 const std::vector<const TokenId*>* mapped) {
    if (!memo_.slots) mapped = nullptr;  // the plain path stages with copy kernels
    // Tokens, chain descriptors and digests live in mapped pinned memory and
    // move by SM loads/stores, so a lookup never queues on the copy engines
    // behind in-flight KV transfers.
    // each chain starts on a 16-byte boundary (vector loads of full rows)
    h_tokens_.reserve(grow((total_tokens + 4 * seqs.size()) * sizeof(TokenId) + 64));
    h_chains_.reserve(grow(seqs.size() * sizeof(ChainDesc)));
    h_out_.reserve(grow(total_chunks * 32));
    auto* tok = reinterpret_cast<TokenId*>(h_tokens_.host);
    auto* ch = reinterpret_cast<ChainDesc*>(h_chains_.host);
    size_t toff = 0, row = 0;
    unsigned long long* srcs = nullptr;
    if (mapped) {  // the fingerprint pass reads each prompt where it already is
        h_srcs_.reserve(grow(seqs.size() * sizeof(unsigned long long)));
        srcs = reinterpret_cast<unsigned long long*>(h_srcs_.host);
    }
    for (size_t i = 0; i < seqs.size(); ++i) {
        toff = (toff + 3) & ~size_t(3);
        if (mapped)
            srcs[i] = reinterpret_cast<unsigned long long>((*mapped)[i]);
        else
            host_copy(tok + toff, seqs[i].data(), seqs[i].size() * sizeof(TokenId));
        ChainDesc d;
        d.token_off = toff;
        d.n_tokens = uint32_t(seqs[i].size());
        d.out_first = uint32_t(row);
        if (parents) std::copy((*parents)[i].begin(), (*parents)[i].end(), d.parent);
        ch[i] = d;
        toff += seqs[i].size();
        row += (seqs[i].size() + chunk_size_ - 1) / chunk_size_;
    }
    p.chunk_size = uint32_t(chunk_size_);
    p.tag_len = uint32_t(tag_.size());
    std::copy(tag_.begin(), tag_.end(), p.tag);

    const size_t tok_bytes = toff * sizeof(TokenId);
    const size_t ch_bytes = seqs.size() * sizeof(ChainDesc);
    d_tokens_.reserve(grow(tok_bytes + 64));
    d_chains_.reserve(grow(ch_bytes + 64));
    if (d_out_.bytes < total_chunks * 32) {
        d_out_.reserve(grow(total_chunks * 32));
        // rows past a chain's first absent chunk are never hashed, but the
        // verify pass copies every row out (the host reads only the hashed
        // ones): defined bytes, not stale allocations
        TKV_CUDA(cudaMemsetAsync(d_out_.ptr, 0, d_out_.bytes, stream_));
    }
    h_bad_.reserve(grow(seqs.size() * sizeof(unsigned int)));
    h_first_.reserve(grow(seqs.size() * sizeof(uint32_t)));
    auto* bad = reinterpret_cast<unsigned int*>(h_bad_.host);
    std::fill(bad, bad + seqs.size(), ~0u);
    MemoView m = memo_;
    if (memo_.slots) {
        // memo_used_bound_ bounds the links inserted so far; resetting here,
        // before the probe, never invalidates a hit this call relies on.
        if (memo_used_bound_ + max_inserts > memo_.entry_cap) memo_reset_locked();
        memo_used_bound_ += max_inserts;
        d_hit_.reserve(grow(total_chunks * sizeof(uint32_t)));
        d_keys_.reserve(grow(total_chunks * sizeof(unsigned long long)));
        d_first_.reserve(grow(seqs.size() * sizeof(uint32_t)));
        m = memo_;
        m.hit_entry = reinterpret_cast<uint32_t*>(d_hit_.ptr);
        m.keys = reinterpret_cast<unsigned long long*>(d_keys_.ptr);
        m.first_miss = reinterpret_cast<uint32_t*>(d_first_.ptr);
    }
    if (memo_.slots) {  // descriptors + token staging + per-row fingerprints in one pass
        TKV_CUDA(launch_memo_stage_chains(reinterpret_cast<const uint32_t*>(h_tokens_.dev),
                                          reinterpret_cast<uint32_t*>(d_tokens_.ptr),
                                          reinterpret_cast<const ChainDesc*>(h_chains_.dev),
                                          reinterpret_cast<ChainDesc*>(d_chains_.ptr), uint32_t(seqs.size()),
                                          uint32_t(total_chunks), p, m, stream_,
                                          mapped ? reinterpret_cast<const unsigned long long*>(h_srcs_.dev)
                                                 : nullptr));
    } else {
        TKV_CUDA(launch_sm_copy(h_chains_.dev, d_chains_.ptr, ch_bytes, stream_));
        TKV_CUDA(launch_sm_copy(h_tokens_.dev, d_tokens_.ptr, tok_bytes, stream_));
    }
    return m;
}

// Re-hashes, without the memo, the chains whose memo hits failed
// verification (first_bad != ~0: a 40-bit tag collision), from the first bad
// chunk on, and republishes every row. Caller holds mu_.
void KeyHasher::rehash_bad_locked(size_t n_chains, size_t total_chunks, const HashParams& p) {
    auto* bad = reinterpret_cast<unsigned int*>(h_bad_.host);
    auto* ch = reinterpret_cast<ChainDesc*>(h_chains_.host);
    std::vector<ChainDesc> redo;
    for (size_t i = 0; i < n_chains; ++i) {
        if (bad[i] == ~0u) continue;
        ChainDesc d = ch[i];
        const size_t skip = size_t(bad[i]) * chunk_size_;
        d.token_off += skip;
        d.n_tokens -= uint32_t(skip);
        d.out_first += bad[i];
        if (bad[i]) std::copy(h_out_.host + 32 * (d.out_first - 1), h_out_.host + 32 * d.out_first, d.parent);
        redo.push_back(d);
        bad[i] = ~0u;
    }
    if (redo.empty()) return;
    ++memo_rehashes_;
    // the redo descriptors go after the launch's own (d_chains_ keeps those)
    std::vector<ChainDesc> all(ch, ch + n_chains);
    all.insert(all.end(), redo.begin(), redo.end());
    h_chains_.reserve(grow(all.size() * sizeof(ChainDesc)));
    d_chains_.reserve(grow(all.size() * sizeof(ChainDesc) + 64));
    ch = reinterpret_cast<ChainDesc*>(h_chains_.host);
    std::copy(all.begin(), all.end(), ch);
    TKV_CUDA(launch_sm_copy(h_chains_.dev, d_chains_.ptr, all.size() * sizeof(ChainDesc), stream_));
    const auto* d_tok = reinterpret_cast<const uint32_t*>(d_tokens_.ptr);
    const auto* d_ch = reinterpret_cast<const ChainDesc*>(d_chains_.ptr);
    TKV_CUDA(launch_hash_chains(d_tok, d_ch + n_chains, uint32_t(redo.size()), p, d_out_.ptr, stream_, nullptr));
    TKV_CUDA(launch_memo_verify(d_tok, d_ch, uint32_t(n_chains), uint32_t(total_chunks), p, d_out_.ptr, nullptr,
                                h_out_.dev, nullptr, stream_));
    TKV_CUDA(cudaStreamSynchronize(stream_));
}

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
    HashParams p;
    MemoView m = stage_locked(seqs, parents, total_tokens, total_chunks, total_chunks, p);
    const double t_packed = trace_lookup() ? now_us() : 0;
    // Run the chains writing digests to HBM, then verify memo hits and
    // publish every digest to the mapped result buffer.
    const auto* d_tok = reinterpret_cast<const uint32_t*>(d_tokens_.ptr);
    const auto* d_ch = reinterpret_cast<const ChainDesc*>(d_chains_.ptr);
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
    rehash_bad_locked(seqs.size(), total_chunks, p);

    size_t row = 0;
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

void KeyHasher::enable_presence(size_t max_entries, PresenceDrain drain) {
    std::lock_guard lock(mu_);
    TKV_CUDA(cudaSetDevice(device_));
    size_t cap = 1024;
    while (cap < 4 * max_entries) cap <<= 1;
    presence_table_.reserve(cap * 64);
    TKV_CUDA(cudaMemsetAsync(presence_table_.ptr, 0, cap * 64, stream_));
    witness_table_.reserve(cap * 16);
    witness_meta_.reserve(64);
    TKV_CUDA(cudaMemsetAsync(witness_table_.ptr, 0, cap * 16, stream_));
    TKV_CUDA(cudaMemsetAsync(witness_meta_.ptr, 0, 64, stream_));
    TKV_CUDA(cudaStreamSynchronize(stream_));
    presence_mask_ = uint32_t(cap - 1);
    presence_used_ = 0;
    presence_drain_ = std::move(drain);
}

// The tier's pending presence changes into this launch's MemoView (applied
// by its first kernel). A table that would fill past half its slots with
// entries and tombstones is cleared and reloaded from a full snapshot.
// Caller holds mu_.
void KeyHasher::presence_sync_locked(MemoView& m) {
    bool reset = false;
    presence_drain_(false, presence_pending_, reset);
    size_t adds = 0;
    for (const auto& u : presence_pending_) adds += u.second;
    const size_t cap = size_t(presence_mask_) + 1;
    if (!reset && presence_used_ + adds > cap / 2) {
        presence_drain_(true, presence_pending_, reset);  // everything present, from scratch
        adds = presence_pending_.size();
    }
    if (reset) {
        TKV_CUDA(cudaMemsetAsync(presence_table_.ptr, 0, cap * 64, stream_));
        TKV_CUDA(cudaMemsetAsync(witness_table_.ptr, 0, cap * 16, stream_));
        TKV_CUDA(cudaMemsetAsync(witness_meta_.ptr, 0, 64, stream_));
        presence_used_ = 0;
    }
    presence_used_ += adds;
    const size_t n = presence_pending_.size();
    h_updates_.reserve(grow(std::max<size_t>(1, n) * 36));
    auto* w = reinterpret_cast<uint32_t*>(h_updates_.host);
    for (size_t i = 0; i < n; ++i) {
        std::memcpy(w + 9 * i, presence_pending_[i].first.data(), 32);
        w[9 * i + 8] = presence_pending_[i].second ? 1u : 0u;
    }
    m.presence.slots = reinterpret_cast<uint32_t*>(presence_table_.ptr);
    m.presence.mask = presence_mask_;
    m.presence.updates = reinterpret_cast<const uint32_t*>(h_updates_.dev);
    m.presence.n_updates = uint32_t(n);
    // the absence witness needs the memo's link index (TKV_NO_WITNESS: off)
    static const bool no_witness = std::getenv("TKV_NO_WITNESS") != nullptr;
    const bool witness = memo_.links != nullptr && !no_witness;
    m.presence.witness = witness ? reinterpret_cast<unsigned long long*>(witness_table_.ptr) : nullptr;
    m.presence.unknown = witness ? reinterpret_cast<unsigned int*>(witness_meta_.ptr) : nullptr;
    m.presence.links = memo_.links;
    m.presence.link_mask = memo_.link_mask;
}

// Cold-lookup fast path: row 0 of every chain in one launch (first_row
// kernel) reading its tokens from mapped memory; the host spins on the
// published flags. True (and `out` / `present_rows` filled) when every
// chain's first chunk is absent: the stored prefix is then empty everywhere
// and nothing else needs hashing. Caller holds mu_.
bool KeyHasher::first_row_lookup(const std::vector<TokenSpanView>& seqs, const std::vector<size_t>& rows,
                                 std::vector<std::vector<Digest>>& out, std::vector<size_t>& present_rows,
                                 const std::function<void()>& while_waiting, bool& waited) {
    const size_t n_chains = seqs.size();
    const double t_pack0 = trace_lookup() ? now_us() : 0;
    h_row0_tok_.reserve(grow(n_chains * chunk_size_ * sizeof(TokenId) + 64));
    h_row0_ch_.reserve(grow(n_chains * sizeof(ChainDesc)));
    h_row0_out_.reserve(grow(n_chains * 36 + n_chains * 32 + 64));
    auto* tok = reinterpret_cast<TokenId*>(h_row0_tok_.host);
    auto* ch = reinterpret_cast<ChainDesc*>(h_row0_ch_.host);
    auto* dig = reinterpret_cast<uint32_t*>(h_row0_out_.host);
    auto* flags = dig + 8 * n_chains;
    for (size_t i = 0; i < n_chains; ++i) {
        const size_t n = std::min(chunk_size_, seqs[i].size());
        std::copy(seqs[i].begin(), seqs[i].begin() + n, tok + i * chunk_size_);
        ChainDesc d;
        d.token_off = i * chunk_size_;
        d.n_tokens = uint32_t(n);
        d.out_first = uint32_t(i);
        ch[i] = d;
        std::atomic_ref<uint32_t>(flags[i]).store(0, std::memory_order_relaxed);
    }
    HashParams p;
    p.chunk_size = uint32_t(chunk_size_);
    p.tag_len = uint32_t(tag_.size());
    std::copy(tag_.begin(), tag_.end(), p.tag);
    if (memo_used_bound_ + n_chains > memo_.entry_cap) memo_reset_locked();
    memo_used_bound_ += n_chains;  // one link per chain at most
    FirstRowInline one;
    const bool inline_one = n_chains == 1;
    if (inline_one) {
        one.n = uint32_t(std::min(chunk_size_, seqs[0].size()));
        std::copy(seqs[0].begin(), seqs[0].begin() + one.n, one.tok);
    }
    TKV_CUDA(launch_first_row(reinterpret_cast<const uint32_t*>(h_row0_tok_.dev),
                              reinterpret_cast<const ChainDesc*>(h_row0_ch_.dev), uint32_t(n_chains), p, memo_,
                              reinterpret_cast<uint32_t*>(h_row0_out_.dev), reinterpret_cast<uint32_t*>(h_row0_out_.dev) +
                              8 * n_chains, stream_,
                              trace_lookup() ? reinterpret_cast<unsigned long long*>(
                                                   h_row0_out_.dev + ((n_chains * 36 + 7) / 8) * 8)
                                             : nullptr,
                              inline_one ? &one : nullptr));
    memo_.presence.n_updates = 0;  // applied by that launch (one CTA) or the separate launch before it
    const double t_launched = trace_lookup() ? now_us() : 0;
    if (while_waiting) {  // the caller's host work runs under the kernel
        while_waiting();
        waited = true;
    }
    const double t_waited = trace_lookup() ? now_us() : 0;
    // spin on the flags (a few tens of microseconds); a synchronize surfaces
    // a failed launch instead of spinning forever
    const double t0 = now_us();
    for (size_t i = 0; i < n_chains;) {
        if (std::atomic_ref<uint32_t>(flags[i]).load(std::memory_order_acquire) != 0) {
            ++i;
        } else if (now_us() - t0 > 2000.0) {
            TKV_CUDA(cudaStreamSynchronize(stream_));
            for (size_t j = i; j < n_chains; ++j)
                if (std::atomic_ref<uint32_t>(flags[j]).load(std::memory_order_acquire) == 0)
                    throw CudaError("first-row lookup kernel published no result");
            break;
        }
    }
    chunks_ += n_chains;
    if (trace_lookup()) {
        TKV_CUDA(cudaStreamSynchronize(stream_));
        const auto* tr = reinterpret_cast<const unsigned long long*>(h_row0_out_.host + ((n_chains * 36 + 7) / 8) * 8);
        std::fprintf(stderr, "[tkv first-row] pack+launch=%.1fus host-work=%.1fus spin=%.1fus | device: staged %.1fus "
                     "hashed %.1fus published %.1fus\n", t_launched - t_pack0, t_waited - t_launched,
                     now_us() - t_waited, (tr[1] - tr[0]) / 1e3, (tr[2] - tr[1]) / 1e3, (tr[3] - tr[2]) / 1e3);
    }
    for (size_t i = 0; i < n_chains; ++i)
        if (rows[i] > 0 && (flags[i] & 2u)) return false;  // a first chunk is stored: the full lookup
    ++launches_;  // the lookup's one hash pass (a fall-through counts the full pass instead)
    for (size_t i = 0; i < n_chains; ++i) {
        present_rows[i] = 0;
        out[i].clear();
        if (rows[i] == 0 || (flags[i] & 4u)) continue;  // (4: absent by the witness, not hashed)
        Digest d;
        std::memcpy(d.data(), dig + 8 * i, 32);
        out[i].push_back(d);
    }
    return true;
}

std::vector<std::vector<Digest>> KeyHasher::hash_prefix(const std::vector<TokenSpanView>& seqs,
                                                        const PresentPrefix& present,
                                                        const std::function<void()>& while_waiting,
                                                        std::vector<size_t>* present_rows,
                                                        const std::vector<const TokenId*>* mapped) {
    const double t_in = trace_lookup() ? now_us() : 0;
    std::lock_guard lock(mu_);
    const double t_locked = trace_lookup() ? now_us() : 0;
    TKV_CUDA(cudaSetDevice(device_));
    const size_t n_chains = seqs.size();
    size_t total_tokens = 0, total_chunks = 0;
    std::vector<size_t> rows(n_chains), first_row(n_chains);
    for (size_t i = 0; i < n_chains; ++i) {
        first_row[i] = total_chunks;
        rows[i] = (seqs[i].size() + chunk_size_ - 1) / chunk_size_;
        total_tokens += seqs[i].size();
        total_chunks += rows[i];
    }
    std::vector<std::vector<Digest>> out(n_chains);
    if (present_rows) present_rows->assign(n_chains, 0);
    if (total_chunks == 0) {
        if (while_waiting) while_waiting();
        return out;
    }
    HashParams p;
    const bool on_device = memo_.slots != nullptr && presence_drain_ && present_rows != nullptr;
    bool waited = false;  // while_waiting already ran (during the first-row kernel)
    // Route: a prompt whose first chunk this hasher has seen before (a host
    // hint set of row-0 token hashes) goes straight to the full lookup — its
    // prefix is most likely stored; a new one first asks the first-row kernel,
    // which answers a cold prompt in one launch. Either route gives the same
    // result; the hint only picks the faster one.
    bool novel = false;
    std::vector<uint64_t> row0(n_chains);
    for (size_t i = 0; i < n_chains; ++i) {
        // the first chunk's tokens only (prompts sharing a document differ after it)
        const size_t m = std::min(chunk_size_, seqs[i].size());
        uint64_t h = 0x9e3779b97f4a7c15ull ^ m;
        for (size_t j = 0; j < m; ++j) h = (h ^ seqs[i][j]) * 0x100000001b3ull;
        row0[i] = h ^ (h >> 29);
        novel |= rows[i] > 0 && seen_row0_.count(row0[i]) == 0;
    }
    if (seen_row0_.size() > (1u << 20)) seen_row0_.clear();
    for (uint64_t h : row0) seen_row0_.insert(h);
    const bool use_first_row = on_device && novel && chunk_size_ <= 256 && std::getenv("TKV_NO_FIRST_ROW") == nullptr;
    const double t_hinted = trace_lookup() ? now_us() : 0;
    if (on_device) {
        // The tier's changes since the last lookup, applied by this lookup's
        // first kernel (the first-row kernel when it is one CTA, else the
        // fingerprint pass) or, for a multi-CTA first-row launch, by a
        // separate launch before it.
        const double ts0 = trace_lookup() ? now_us() : 0;
        presence_sync_locked(memo_);
        const uint32_t n_upd = memo_.presence.n_updates;
        // a multi-CTA first-row launch, or more changes than its apply warps
        // take in one round (each change probes the link index and the
        // witness): the whole grid applies them first
        if (use_first_row && (n_chains > 2 || n_upd > 192)) {
            TKV_CUDA(launch_presence_apply(memo_.presence, stream_));
            memo_.presence.n_updates = 0;
        }
        if (trace_lookup())
            std::fprintf(stderr, "[tkv presence] changes=%u sync=%.1fus | lock=%.1fus route=%.1fus\n", n_upd,
                         now_us() - ts0, t_locked - t_in, t_hinted - t_locked);
    }
    if (use_first_row && first_row_lookup(seqs, rows, out, *present_rows, while_waiting, waited)) {
        if (trace_lookup())
            std::fprintf(stderr, "[tkv prefix] chains=%zu first-row decided in %.1fus\n", n_chains, now_us() - t_in);
        return out;  // every first chunk absent: decided without staging the prompts
    }
    // the first launch inserts at most one link per chain; the prompts are
    // read in place when the caller's mapped copies are already filled (the
    // first-row route); otherwise they are packed here and the caller's copy
    // runs under the kernels (filling the mapped copies first and skipping
    // the pack measured no faster: the device work is then exposed instead)
    const double t_routed = trace_lookup() ? now_us() : 0;
    MemoView m = stage_locked(seqs, nullptr, total_tokens, total_chunks, n_chains, p, waited ? mapped : nullptr);
    memo_.presence.n_updates = 0;  // applied by the fingerprint pass (or the first-row kernel)
    auto* dev_present = reinterpret_cast<uint32_t*>(h_present_.host);
    auto* dev_known = reinterpret_cast<uint32_t*>(h_known_.host);
    if (on_device) {
        h_present_.reserve(grow(n_chains * sizeof(uint32_t)));
        h_known_.reserve(grow(n_chains * sizeof(uint32_t)));
        dev_present = reinterpret_cast<uint32_t*>(h_present_.host);
        dev_known = reinterpret_cast<uint32_t*>(h_known_.host);
        m.lookup.present_out = reinterpret_cast<uint32_t*>(h_present_.dev);
        m.lookup.known_out = reinterpret_cast<uint32_t*>(h_known_.dev);
    } else {
        m.presence = PresenceView{};
    }
    const double t_packed = trace_lookup() ? now_us() : 0;
    const auto* d_tok = reinterpret_cast<const uint32_t*>(d_tokens_.ptr);
    const auto* d_ch = reinterpret_cast<const ChainDesc*>(d_chains_.ptr);
    auto* first = reinterpret_cast<uint32_t*>(h_first_.host);
    auto* bad = reinterpret_cast<unsigned int*>(h_bad_.host);
    std::vector<size_t> known(n_chains, 0);
    ++launches_;
    // 1. every row probed at once (memo), the first row past the hits of
    //    every chain hashed (one SHA chunk: the reference's
    //    longest_prefix_match also stops at the first absent chunk,
    //    tokens.cpp:59-69), the hits verified exactly, all in one round trip.
    m.max_rows = 1;
    TKV_CUDA(launch_hash_chains(d_tok, d_ch, uint32_t(n_chains), p, d_out_.ptr, stream_, &m));
    MemoView vm = m;
    vm.first_miss_out = reinterpret_cast<uint32_t*>(h_first_.dev);
    TKV_CUDA(launch_memo_verify(d_tok, d_ch, uint32_t(n_chains), uint32_t(total_chunks), p, d_out_.ptr,
                                memo_.slots ? &vm : nullptr, h_out_.dev,
                                reinterpret_cast<unsigned int*>(h_bad_.dev), stream_));
    if (while_waiting && !waited) while_waiting();
    const double t_launched = trace_lookup() ? now_us() : 0;
    TKV_CUDA(cudaStreamSynchronize(stream_));
    const double t_synced = trace_lookup() ? now_us() : 0;
    int passes = 0;
    std::vector<bool> decided(n_chains, false);
    for (size_t i = 0; i < n_chains; ++i) {
        if (on_device && bad[i] == ~0u && (dev_present[i] & 0x80000000u)) {
            // the device decided: memo hits verified, presence from the index
            decided[i] = true;
            known[i] = dev_known[i];
            (*present_rows)[i] = dev_present[i] & 0x7fffffffu;
            continue;
        }
        const size_t f = memo_.slots ? size_t(first[i]) : 0;
        known[i] = std::min(rows[i], f + 1);
        if (memo_.slots && bad[i] != ~0u) known[i] = std::min<size_t>(known[i], bad[i]);
    }
    // 2. the leading present chunks: a chain whose known chunks are all
    //    present (a memo that lost its links, or a failed hit) continues —
    //    one chunk at a time is the reference's order; here the first pass
    //    adds one chunk and the second hashes the rest in one launch.
    auto digests_of = [&](size_t i, size_t n) {
        std::vector<Digest> d(n);
        for (size_t c = 0; c < n; ++c)
            std::copy(h_out_.host + 32 * (first_row[i] + c), h_out_.host + 32 * (first_row[i] + c) + 32,
                      d[c].begin());
        return d;
    };
    auto ch = reinterpret_cast<const ChainDesc*>(h_chains_.host);
    for (int pass = 0; pass < 2; ++pass) {
        // (a chain with a failed memo hit re-enters here one chunk at a time)
        std::vector<ChainDesc> more;
        std::vector<size_t> which;
        for (size_t i = 0; i < n_chains; ++i) {
            if (decided[i] || known[i] >= rows[i]) continue;
            const auto d = digests_of(i, known[i]);
            if (present(d) < known[i]) continue;  // the LPM ended inside the hits
            ChainDesc x = ch[i];
            const size_t skip = known[i] * chunk_size_;
            x.token_off += skip;
            x.n_tokens = pass == 0 ? uint32_t(std::min(chunk_size_, seqs[i].size() - skip))
                                   : uint32_t(seqs[i].size() - skip);
            x.out_first = uint32_t(first_row[i] + known[i]);
            if (known[i]) std::copy(d[known[i] - 1].begin(), d[known[i] - 1].end(), x.parent);
            more.push_back(x);
            which.push_back(i);
        }
        if (more.empty()) break;
        ++passes;
        std::vector<ChainDesc> all(ch, ch + n_chains);
        all.insert(all.end(), more.begin(), more.end());
        h_chains_.reserve(grow(all.size() * sizeof(ChainDesc)));
        d_chains_.reserve(grow(all.size() * sizeof(ChainDesc) + 64));
        std::copy(all.begin(), all.end(), reinterpret_cast<ChainDesc*>(h_chains_.host));
        ch = reinterpret_cast<const ChainDesc*>(h_chains_.host);
        d_ch = reinterpret_cast<const ChainDesc*>(d_chains_.ptr);
        TKV_CUDA(launch_sm_copy(h_chains_.dev, d_chains_.ptr, all.size() * sizeof(ChainDesc), stream_));
        MemoView ins = m;  // insert the new links under their full-prefix keys
        ins.first_miss = nullptr;
        ins.max_rows = 0;  // the descriptors bound the rows
        ins.lookup = LookupOut{};
        // no reset mid-call (the hits above point into the memo): links past
        // the capacity are simply not inserted (memo_insert checks it)
        for (const auto& x : more) memo_used_bound_ += (x.n_tokens + chunk_size_ - 1) / chunk_size_;
        TKV_CUDA(launch_hash_chains(d_tok, d_ch + n_chains, uint32_t(more.size()), p, d_out_.ptr, stream_,
                                    memo_.slots ? &ins : nullptr));
        TKV_CUDA(launch_memo_verify(d_tok, d_ch, uint32_t(n_chains), uint32_t(total_chunks), p, d_out_.ptr,
                                    nullptr, h_out_.dev, nullptr, stream_));
        TKV_CUDA(cudaStreamSynchronize(stream_));
        for (size_t k = 0; k < which.size(); ++k) {
            const size_t i = which[k];
            chunks_ += more[k].n_tokens ? (more[k].n_tokens + chunk_size_ - 1) / chunk_size_ : 0;
            known[i] = pass == 0 ? known[i] + 1 : rows[i];
        }
    }
    for (size_t i = 0; i < n_chains; ++i) {
        out[i] = digests_of(i, known[i]);
        if (present_rows && !decided[i]) {
            (*present_rows)[i] = present(out[i]);
            ++host_decided_;
        }
    }
    if (trace_lookup())
        std::fprintf(stderr, "[tkv prefix] chains=%zu rows=%zu pre=%.1fus pack=%.1fus launch=%.1fus "
                     "device+sync=%.1fus passes=%d rest=%.1fus\n", n_chains, total_chunks, t_routed - t_in,
                     t_packed - t_routed, t_launched - t_packed, t_synced - t_launched, passes, now_us() - t_synced);
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
    link_table_.reserve(slots * 64);  // one link per entry at most, half full at worst
    memo_.links = reinterpret_cast<uint32_t*>(link_table_.ptr);
    memo_.link_mask = uint32_t(slots - 1);
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
    // the links go too: present digests added from now on without a link are
    // counted unknown (the witness is then off until they leave the tier);
    // those already counted keep their key in the presence slot
    if (memo_.links) TKV_CUDA(cudaMemsetAsync(memo_.links, 0, (size_t(memo_.link_mask) + 1) * 64, stream_));
    memo_used_bound_ = 0;
    ++memo_resets_;
}

KeyHasher::MemoStats KeyHasher::memo_stats() {
    std::lock_guard lock(mu_);
    MemoStats s;
    if (!memo_.slots) return s;
    unsigned long long st[3] = {0, 0, 0};
    TKV_CUDA(cudaMemcpyAsync(st, memo_.stats, sizeof st, cudaMemcpyDeviceToHost, stream_));
    TKV_CUDA(cudaStreamSynchronize(stream_));
    s.hits = st[0];
    s.misses = st[1];
    s.capacity = memo_.entry_cap;
    s.resets = memo_resets_ - 1;  // the enabling clear is not a reset
    s.rehashes = memo_rehashes_;
    s.witnessed = st[2];
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
