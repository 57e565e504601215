#include "store.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "record.hpp"

namespace tkv {

const Status& PutHandle::wait() const {
    std::unique_lock lock(st_->m);
    st_->cv.wait(lock, [&] { return st_->done; });
    return st_->status;
}

bool PutHandle::done() const {
    std::lock_guard lock(st_->m);
    return st_->done;
}

PutHandle PutHandle::immediate(Status st) {
    auto s = std::make_shared<detail::PutState>();
    s->done = true;
    s->status = std::move(st);
    return PutHandle(s);
}

namespace {
void finish(const std::shared_ptr<detail::PutState>& s, Status st) {
    {
        std::lock_guard lock(s->m);
        s->status = std::move(st);
        s->done = true;
    }
    s->cv.notify_all();
}
}  // namespace

size_t TieredStore::presence_subscribe() {
    std::lock_guard lock(mu_);
    feeds_.push_back(std::make_unique<PresenceFeed>());
    return feeds_.size() - 1;
}

void TieredStore::PresenceFeed::note(const Digest& d, bool present) {
    if (index.size() < 2 * (pending.size() + 1)) {  // grow (a power of two) and re-index
        size_t cap = 1024;
        while (cap < 4 * (pending.size() + 1)) cap <<= 1;
        index.assign(cap, -1);
        const size_t mask = index.size() - 1;
        for (size_t k = 0; k < pending.size(); ++k) {
            uint64_t h;
            std::memcpy(&h, pending[k].first.data(), 8);
            size_t i = h & mask;
            while (index[i] >= 0) i = (i + 1) & mask;
            index[i] = int32_t(k);
        }
    }
    const size_t mask = index.size() - 1;
    uint64_t h;
    std::memcpy(&h, d.data(), 8);
    for (size_t i = h & mask;; i = (i + 1) & mask) {
        if (index[i] < 0) {
            index[i] = int32_t(pending.size());
            pending.emplace_back(d, present);
            return;
        }
        if (pending[index[i]].first == d) {
            pending[index[i]].second = present;
            return;
        }
    }
}

void TieredStore::PresenceFeed::clear() {
    pending.clear();
    std::fill(index.begin(), index.end(), -1);
}

void TieredStore::presence_changed(const Digest& d, bool present) {
    const size_t cap = 4 * std::max<size_t>(256, slab_slots());
    for (auto& f : feeds_) {
        if (f->fresh) continue;
        f->note(d, present);
        if (f->pending.size() > cap) {  // a subscriber that stopped draining: resync from a snapshot
            f->clear();
            f->fresh = true;
        }
    }
}

void TieredStore::presence_drain(size_t id, bool want_full, std::vector<std::pair<Digest, bool>>& out,
                                 bool& reset) {
    std::lock_guard lock(mu_);
    PresenceFeed& f = *feeds_.at(id);
    out.clear();
    reset = want_full || f.fresh;
    if (reset) {
        for (const auto& [d, e] : index_)
            if (e.state == Entry::State::present) out.emplace_back(d, true);
        f.fresh = false;
    } else {
        out.swap(f.pending);
    }
    f.clear();
}

TieredStore::TieredStore(StoreConfig cfg) : cfg_(std::move(cfg)) {
    cfg_.model.validate(cfg_.chunk_size);
    slot_bytes_ = cfg_.model.chunk_bytes(cfg_.chunk_size);
    const size_t slots = cfg_.ram_pool_bytes / slot_bytes_;
    // TKV_SLAB_HUGE=0: cudaHostAlloc'ed slab instead of registered huge pages
    // (A/B measurements only).
    const char* hv = std::getenv("TKV_SLAB_HUGE");
    slab_.huge = !(hv && std::strcmp(hv, "0") == 0);
    if (slots) slab_.reserve(slots * slot_bytes_);
    free_slots_.reserve(slots);
    for (size_t i = slots; i > 0; --i) free_slots_.push_back(uint32_t(i - 1));  // slot 0 first
}

TieredStore::~TieredStore() = default;

bool TieredStore::reserve_slot_locked(uint32_t& slot) {
    if (free_slots_.empty()) evict_until_locked(slot_bytes_);
    if (free_slots_.empty()) return false;
    slot = free_slots_.back();
    free_slots_.pop_back();
    return true;
}

// LRU over present, unpinned, unshared entries (store.cpp:198-263, RAM branch).
size_t TieredStore::evict_until_locked(size_t bytes_needed) {
    size_t freed = 0;
    while (freed < bytes_needed) {
        const Digest* victim = nullptr;
        uint64_t oldest = ~uint64_t(0);
        for (const auto& [d, e] : index_) {
            if (e.share_count > 0 || e.state != Entry::State::present || e.pinned) continue;
            if (e.last_touch < oldest) {
                oldest = e.last_touch;
                victim = &d;
            }
        }
        if (!victim) break;
        auto it = index_.find(*victim);
        free_slots_.push_back(it->second.slot);
        presence_changed(it->first, false);
        index_.erase(it);
        freed += slot_bytes_;
    }
    return freed;
}

size_t TieredStore::evict_until(size_t bytes_needed) {
    std::lock_guard lock(mu_);
    return evict_until_locked(bytes_needed);
}

Result<SlotWrite> TieredStore::begin_write(const Digest& digest, uint32_t token_count, bool pin) {
    if (token_count == 0 || token_count > cfg_.chunk_size)
        return Status{Errc::invalid_argument, "chunk geometry does not match store"};
    std::lock_guard lock(mu_);
    auto it = index_.find(digest);
    if (it != index_.end()) {
        Entry& e = it->second;
        if (e.token_count != token_count)
            return Status{Errc::invalid_argument, "digest indexed with other geometry"};
        SlotWrite w;
        if (e.state == Entry::State::present) {
            // Idempotent: already stored, no new bytes (store.cpp:322-329).
            if (pin) e.pinned = true;
            touch(e);
            w.kind = SlotWrite::Kind::already_present;
            w.handle = PutHandle::immediate(Status::success());
        } else {
            w.kind = SlotWrite::Kind::in_flight;
            w.handle = PutHandle(e.writer);
            if (pin) e.pinned = true;
        }
        return w;
    }
    uint32_t slot = 0;
    if (!reserve_slot_locked(slot)) return Status{Errc::tier_full, "ram pool exhausted"};
    Entry e;
    e.state = Entry::State::writing;
    e.token_count = uint16_t(token_count);
    e.slot = slot;
    e.pinned = pin;
    e.writer = std::make_shared<detail::PutState>();
    SlotWrite w;
    w.kind = SlotWrite::Kind::write;
    w.host = slab_.host + size_t(slot) * slot_bytes_;
    w.dev = slab_.dev + size_t(slot) * slot_bytes_;
    w.handle = PutHandle(e.writer);
    index_.emplace(digest, std::move(e));
    return w;
}

std::vector<Result<SlotWrite>> TieredStore::begin_write_batch(
    const std::vector<WriteSpec>& specs, const std::unordered_map<Digest, uint32_t, DigestHasher>& own_shares,
    std::vector<Digest>* touch_order) {
    std::vector<Result<SlotWrite>> out;
    out.reserve(specs.size());
    std::lock_guard lock(mu_);
    std::unordered_map<Digest, size_t, DigestHasher> batch_new;  // written by this batch -> index in out
    // batch_put registers every put (share_count++) before any write runs, so
    // a chunk this batch puts again later stays unevictable until that later
    // put has been applied (store.cpp:455-460).
    std::unordered_map<Digest, uint32_t, DigestHasher> pending;
    for (const auto& s : specs) ++pending[s.digest];
    // Per written output: the largest token count its slot may take (below
    // chunk_size only for the slot of an own-loaded victim with fewer tokens).
    std::vector<std::pair<size_t, uint32_t>> written;
    for (const auto& s : specs) {
        --pending[s.digest];
        if (s.token_count == 0 || s.token_count > cfg_.chunk_size) {
            out.emplace_back(Status{Errc::invalid_argument, "chunk geometry does not match store"});
            continue;
        }
        auto it = index_.find(s.digest);
        if (it != index_.end()) {
            Entry& e = it->second;
            if (e.token_count != s.token_count) {
                out.emplace_back(Status{Errc::invalid_argument, "digest indexed with other geometry"});
                continue;
            }
            SlotWrite w;
            if (s.pin) e.pinned = true;
            if (e.state == Entry::State::present || batch_new.count(s.digest)) {
                touch(e);  // store.cpp:322-329: idempotent put
                if (touch_order) touch_order->push_back(s.digest);
                w.kind = e.state == Entry::State::present ? SlotWrite::Kind::already_present
                                                          : SlotWrite::Kind::in_flight;
                w.handle = e.state == Entry::State::present ? PutHandle::immediate(Status::success())
                                                            : PutHandle(e.writer);
            } else {
                w.kind = SlotWrite::Kind::in_flight;  // an earlier batch is writing it
                w.handle = PutHandle(e.writer);
            }
            out.emplace_back(std::move(w));
            continue;
        }
        uint32_t victim_limit = cfg_.chunk_size;
        if (free_slots_.empty()) {
            const Digest* victim = nullptr;
            uint64_t oldest = ~uint64_t(0);
            for (const auto& [d, e] : index_) {
                if (e.pinned) continue;
                bool cand;
                if (e.state == Entry::State::present) {
                    // An entry this batch is still loading may be overwritten
                    // layer by layer behind its loads (layer l is loaded before
                    // layer l is stored) only if the new chunk's layer l lies
                    // within the old chunk's layers <= l: token_count >= new.
                    auto own = own_shares.find(d);
                    const uint32_t mine = own == own_shares.end() ? 0u : own->second;
                    cand = e.share_count == 0 || (e.share_count <= mine && e.token_count >= s.token_count);
                } else {
                    cand = batch_new.count(d) != 0;
                }
                if (cand) {
                    auto pd = pending.find(d);
                    cand = pd == pending.end() || pd->second == 0;
                }
                if (cand && e.last_touch < oldest) {
                    oldest = e.last_touch;
                    victim = &d;
                }
            }
            if (!victim) {
                out.emplace_back(Status{Errc::tier_full, "ram pool exhausted"});
                continue;
            }
            auto vit = index_.find(*victim);
            auto bn = batch_new.find(vit->first);
            if (bn != batch_new.end()) {  // stored, then evicted, within this batch
                SlotWrite& vw = out[bn->second].value();
                vw.kind = SlotWrite::Kind::dropped;
                vw.host = vw.dev = nullptr;
                finish(vit->second.writer, Status::success());
                batch_new.erase(bn);
            }
            free_slots_.push_back(vit->second.slot);
            if (vit->second.state == Entry::State::present) {
                if (vit->second.share_count) victim_limit = vit->second.token_count;
                presence_changed(vit->first, false);
            }
            index_.erase(vit);
        }
        const uint32_t slot = free_slots_.back();
        free_slots_.pop_back();
        Entry e;
        e.state = Entry::State::writing;
        e.token_count = uint16_t(s.token_count);
        e.slot = slot;
        e.pinned = s.pin;
        e.writer = std::make_shared<detail::PutState>();
        touch(e);  // the reference's write order (replayed at commit)
        if (touch_order) touch_order->push_back(s.digest);
        SlotWrite w;
        w.kind = SlotWrite::Kind::write;
        w.host = slab_.host + size_t(slot) * slot_bytes_;
        w.dev = slab_.dev + size_t(slot) * slot_bytes_;
        w.handle = PutHandle(e.writer);
        batch_new[s.digest] = out.size();
        written.emplace_back(out.size(), victim_limit);
        index_.emplace(s.digest, std::move(e));
        out.emplace_back(std::move(w));
    }
    // Which slot a chunk takes is not part of the outcome (the reference
    // replays only which chunks stay): the full chunks written by this batch
    // take their slots in ascending order, so consecutive chunks land in
    // consecutive slots wherever the freed slots allow and the per-layer
    // host copies go as pitched runs (ce_copy.hpp). Slots limited by an
    // own-loaded victim keep their chunk.
    std::vector<size_t> idx;
    std::vector<uint32_t> slots;
    for (const auto& [o, limit] : written) {
        if (!out[o].ok() || out[o].value().kind != SlotWrite::Kind::write) continue;  // dropped
        if (limit < cfg_.chunk_size || specs[o].token_count != cfg_.chunk_size) continue;
        idx.push_back(o);
        slots.push_back(index_.at(specs[o].digest).slot);
    }
    if (idx.size() > 1 && !std::is_sorted(slots.begin(), slots.end())) {
        std::sort(slots.begin(), slots.end());
        for (size_t k = 0; k < idx.size(); ++k) {
            SlotWrite& w = out[idx[k]].value();
            index_.at(specs[idx[k]].digest).slot = slots[k];
            w.host = slab_.host + size_t(slots[k]) * slot_bytes_;
            w.dev = slab_.dev + size_t(slots[k]) * slot_bytes_;
        }
    }
    return out;
}

void TieredStore::commit_batch(const std::vector<Digest>& digests, const std::vector<Digest>& touches) {
    // Everything under one lock, and the writers finished only afterwards:
    // whoever waits on a put handle then sees the batch's final LRU order.
    std::vector<std::shared_ptr<detail::PutState>> writers;
    {
        std::lock_guard lock(mu_);
        for (const auto& d : digests) {
            auto it = index_.find(d);
            if (it == index_.end() || it->second.state != Entry::State::writing) continue;
            writers.push_back(std::move(it->second.writer));
            it->second.state = Entry::State::present;
            presence_changed(d, true);
            touch(it->second);
        }
        for (const auto& d : touches) {
            auto it = index_.find(d);
            if (it != index_.end()) touch(it->second);
        }
    }
    for (auto& w : writers)
        if (w) finish(w, Status::success());
}

void TieredStore::commit_write(const Digest& digest, const Status& status) {
    std::shared_ptr<detail::PutState> writer;
    {
        std::lock_guard lock(mu_);
        auto it = index_.find(digest);
        if (it == index_.end() || it->second.state != Entry::State::writing) return;
        writer = std::move(it->second.writer);
        if (status.ok()) {
            it->second.state = Entry::State::present;
            presence_changed(digest, true);
            touch(it->second);
        } else {
            free_slots_.push_back(it->second.slot);
            index_.erase(it);
        }
    }
    if (writer) finish(writer, status);
}

Result<SlotRead> TieredStore::acquire(const Digest& digest, uint32_t expect_tokens) {
    std::lock_guard lock(mu_);
    auto it = index_.find(digest);
    if (it == index_.end() || it->second.state != Entry::State::present)
        return Status{Errc::not_found, "no such chunk"};
    Entry& e = it->second;
    if (expect_tokens && e.token_count != expect_tokens)
        return Status{Errc::size_mismatch, "record token count differs from plan"};
    e.share_count++;
    touch(e);
    return SlotRead{slab_.host + size_t(e.slot) * slot_bytes_,
                    slab_.dev + size_t(e.slot) * slot_bytes_, e.token_count};
}

void TieredStore::release(const Digest& digest) {
    std::lock_guard lock(mu_);
    auto it = index_.find(digest);
    if (it != index_.end() && it->second.share_count > 0) it->second.share_count--;
}

PutHandle TieredStore::put(const Digest& digest, uint32_t token_count, const uint8_t* payload,
                           size_t payload_bytes, bool pin) {
    if (payload_bytes != size_t(token_count) * cfg_.model.num_layers *
                             cfg_.model.bytes_per_token_per_layer)
        return PutHandle::immediate(Status{Errc::invalid_argument, "chunk geometry does not match store"});
    auto w = begin_write(digest, token_count, pin);
    if (!w.ok()) return PutHandle::immediate(w.status());
    if (w.value().kind != SlotWrite::Kind::write) return w.value().handle;
    std::memcpy(w.value().host, payload, payload_bytes);
    commit_write(digest, Status::success());
    return w.value().handle;
}

Result<std::vector<uint8_t>> TieredStore::get(const Digest& digest) {
    auto r = acquire(digest, 0);
    if (!r.ok()) return r.status();
    const size_t n = size_t(r.value().token_count) * cfg_.model.num_layers *
                     cfg_.model.bytes_per_token_per_layer;
    std::vector<uint8_t> out(r.value().host, r.value().host + n);
    release(digest);
    return out;
}

Result<std::vector<uint8_t>> TieredStore::get_layer(const Digest& digest, uint32_t layer) {
    // store.cpp:654-680: an absent chunk is not_found before the layer is
    // checked; a present one with a bad layer is invalid_argument (untouched)
    if (layer >= cfg_.model.num_layers)
        return contains(digest) ? Status{Errc::invalid_argument, "layer out of range"}
                                : Status{Errc::not_found, "no such chunk"};
    auto r = acquire(digest, 0);
    if (!r.ok()) return r.status();
    const size_t lb = size_t(r.value().token_count) * cfg_.model.bytes_per_token_per_layer;
    const uint8_t* src = r.value().host + size_t(layer) * lb;
    std::vector<uint8_t> out(src, src + lb);
    release(digest);
    return out;
}

bool TieredStore::contains(const Digest& digest) const {
    std::lock_guard lock(mu_);
    auto it = index_.find(digest);
    return it != index_.end() && it->second.state == Entry::State::present;
}

size_t TieredStore::present_prefix(const std::vector<Digest>& digests) const {
    std::lock_guard lock(mu_);
    size_t k = 0;
    for (; k < digests.size(); ++k) {
        auto it = index_.find(digests[k]);
        if (it == index_.end() || it->second.state != Entry::State::present) break;
    }
    return k;
}

std::vector<bool> TieredStore::present_mask(const std::vector<Digest>& digests) const {
    std::vector<bool> out(digests.size());
    std::lock_guard lock(mu_);
    for (size_t i = 0; i < digests.size(); ++i) {
        auto it = index_.find(digests[i]);
        out[i] = it != index_.end() && it->second.state == Entry::State::present;
    }
    return out;
}

Status TieredStore::pin(const Digest& digest, bool on) {
    std::lock_guard lock(mu_);
    auto it = index_.find(digest);
    if (it == index_.end()) return Status{Errc::not_found, "no such chunk"};
    it->second.pinned = on;
    return Status::success();
}

ClearResult TieredStore::clear(const std::vector<Digest>& digests) {
    ClearResult r;
    std::lock_guard lock(mu_);
    for (const auto& d : digests) {
        auto it = index_.find(d);
        if (it == index_.end()) continue;
        Entry& e = it->second;
        if (e.state != Entry::State::present || e.pinned || e.share_count > 0) {
            r.refused++;
            continue;
        }
        free_slots_.push_back(e.slot);
        presence_changed(d, false);
        index_.erase(it);
        r.removed++;
    }
    return r;
}

Result<std::vector<uint8_t>> TieredStore::export_record(const Digest& digest, uint64_t tag_hash) {
    auto r = acquire(digest, 0);
    if (!r.ok()) return r.status();
    RecordInfo info;
    info.digest = digest;
    info.model_tag_hash = tag_hash;
    info.token_count = uint16_t(r.value().token_count);
    info.num_layers = uint16_t(cfg_.model.num_layers);
    info.bytes_per_token = cfg_.model.bytes_per_token_per_layer;
    auto rec = encode_record(info, r.value().host, info.payload_bytes());
    release(digest);
    return rec;
}

Status TieredStore::export_record_into(const Digest& digest, uint64_t tag_hash, uint8_t* out, size_t cap,
                                      size_t* n) {
    auto r = acquire(digest, 0);
    if (!r.ok()) return r.status();
    RecordInfo info;
    info.digest = digest;
    info.model_tag_hash = tag_hash;
    info.token_count = uint16_t(r.value().token_count);
    info.num_layers = uint16_t(cfg_.model.num_layers);
    info.bytes_per_token = cfg_.model.bytes_per_token_per_layer;
    *n = record_bytes(info.payload_bytes());
    if (out && cap >= *n) encode_record_into(info, r.value().host, info.payload_bytes(), out);
    release(digest);
    return Status::success();
}

Status TieredStore::import_record(const uint8_t* record, size_t n, bool pin) {
    const uint8_t* payload = nullptr;
    auto info = parse_record(record, n, &payload);
    if (!info.ok()) return info.status();
    const auto& i = info.value();
    if (i.num_layers != cfg_.model.num_layers ||
        i.bytes_per_token != cfg_.model.bytes_per_token_per_layer || i.token_count > cfg_.chunk_size)
        return Status{Errc::invalid_argument, "chunk geometry does not match store"};
    return put(i.digest, i.token_count, payload, i.payload_bytes(), pin).wait();
}

StoreStats TieredStore::stats() const {
    std::lock_guard lock(mu_);
    StoreStats s;
    s.entries = index_.size();
    s.ram_slots_total = slot_bytes_ ? slab_.bytes / slot_bytes_ : 0;
    s.ram_slots_used = s.ram_slots_total - free_slots_.size();
    for (const auto& [_, e] : index_)
        if (e.state == Entry::State::present) s.ram_entries++;
    return s;
}

}  // namespace tkv
