// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference tierkv sources (compiled in place
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets
// the Python tests and bench.py's CPU-baseline arm drive the reference's own
// public API — tokens.hpp, paged_store.hpp, store.hpp, connector.hpp,
// pd_staging.hpp, synth.hpp — exactly the way the reference tests do
// (tests/test_connector.cpp:51-178), so both engines can be run on identical
// inputs and compared byte for byte.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "tierkv/chunk_file.hpp"
#include "tierkv/codec.hpp"
#include "tierkv/connector.hpp"
#include "tierkv/hash.hpp"
#include "tierkv/paged_store.hpp"
#include "tierkv/pd_staging.hpp"
#include "tierkv/store.hpp"
#include "tierkv/synth.hpp"
#include "tierkv/tokens.hpp"

using namespace tierkv;

namespace {

struct RefEngine {
    StoreConfig scfg;
    std::unique_ptr<TieredStore> store;
    std::unique_ptr<PagedKVStore> pages;
    std::unique_ptr<Connector> conn;
    std::vector<ConnectorMetadata> metas;
};

ModelSpec make_spec(uint32_t layers, uint32_t bpt, uint32_t page_tokens, const char* tag) {
    ModelSpec s;
    s.num_layers = layers;
    s.bytes_per_token_per_layer = bpt;
    s.page_tokens = page_tokens;
    s.model_tag = tag;
    return s;
}

}  // namespace

extern "C" {

// --- tokens.hpp / hash.hpp / synth.hpp -------------------------------------

// tokens.cpp:49-57. Writes n_chunks * 32 digest bytes; returns n_chunks.
size_t ref_chunk_keys(const uint32_t* tokens, size_t n, size_t chunk_size, const char* tag,
                      uint8_t* out) {
    auto keys = chunk_keys(TokenSpanView(tokens, n), chunk_size, tag);
    for (size_t i = 0; i < keys.size(); ++i) std::memcpy(out + 32 * i, keys[i].digest.data(), 32);
    return keys.size();
}

// KeyChain::reset + next (tokens.cpp:22-47): one link from an explicit parent.
void ref_keychain_next(const uint8_t* parent, uint32_t index, const uint32_t* tokens, size_t n,
                       size_t chunk_size, const char* tag, uint8_t* out) {
    KeyChain chain(tag, chunk_size);
    Digest p;
    std::memcpy(p.data(), parent, 32);
    chain.reset(p, index);
    auto key = chain.next(TokenSpanView(tokens, n));
    std::memcpy(out, key.digest.data(), 32);
}

// tokens.cpp:59-69 with a digest-set KeyIndex (test_tokens.cpp:22-31).
size_t ref_longest_prefix_match(const uint32_t* tokens, size_t n, size_t chunk_size,
                                const char* tag, const uint8_t* digests, size_t n_digests) {
    std::vector<Digest> set(n_digests);
    for (size_t i = 0; i < n_digests; ++i) std::memcpy(set[i].data(), digests + 32 * i, 32);
    KeyIndex index = [&](const ChunkKey& k) {
        for (const auto& d : set)
            if (d == k.digest) return true;
        return false;
    };
    return longest_prefix_match(TokenSpanView(tokens, n), chunk_size, tag, index);
}

void ref_sha256(const uint8_t* data, size_t n, uint8_t* out) {
    Digest d = sha256(ByteSpan(data, n));
    std::memcpy(out, d.data(), 32);
}

uint64_t ref_model_tag_hash(const char* tag) { return model_tag_hash(tag); }
uint64_t ref_fnv1a64(const uint8_t* data, size_t n) { return fnv1a64(ByteSpan(data, n)); }
uint64_t ref_model_seed(const char* tag) {
    ModelSpec s;
    s.model_tag = tag;
    return model_seed_of(s);
}

void ref_synth_layer_kv(uint64_t seed, const uint32_t* tokens, size_t n, uint32_t layer,
                        uint64_t first_pos, uint32_t bpt, uint8_t* out) {
    synth_layer_kv(seed, TokenSpanView(tokens, n), layer, first_pos, bpt,
                   MutByteSpan(out, n * size_t(bpt)));
}

// --- codec.hpp: Q8ScaleCodec ---------------------------------------------------

size_t ref_q8_encode(const uint8_t* payload, size_t n, uint8_t* out) {
    auto blob = q8_scale_codec().encode(ByteSpan(payload, n));
    std::memcpy(out, blob.data(), blob.size());
    return blob.size();
}

// Returns the payload size, or 0 when decode fails (writes Errc to *code).
size_t ref_q8_decode(const uint8_t* blob, size_t n, uint8_t* out, int* code) {
    auto r = q8_scale_codec().decode(ByteSpan(blob, n));
    *code = int(r.code());
    if (!r.ok()) return 0;
    std::memcpy(out, r.value().data(), r.value().size());
    return r.value().size();
}

// --- chunk_file.hpp: LMCK records --------------------------------------------

size_t ref_encode_record(const char* tag, const uint8_t* digest, uint32_t token_count,
                         uint32_t layers, uint32_t bpt, const uint8_t* payload, uint8_t* out) {
    ChunkKey key;
    std::memcpy(key.digest.data(), digest, 32);
    key.model_tag = tag;
    const size_t n = size_t(token_count) * layers * bpt;
    KVChunk c = KVChunk::from_payload(key, token_count, layers, bpt,
                                      std::vector<uint8_t>(payload, payload + n));
    auto rec = encode_chunk_record(c);
    std::memcpy(out, rec.data(), rec.size());
    return rec.size();
}

// Errc of parse_chunk_record (0 = ok); payload copied to out when ok.
int ref_parse_record(const uint8_t* rec, size_t n, uint8_t* out) {
    auto r = parse_chunk_record(ByteSpan(rec, n));
    if (!r.ok()) return int(r.code());
    std::memcpy(out, r.value().payload().data(), r.value().payload().size());
    return 0;
}

// --- engine stack (store + pages + connector) -------------------------------

void* ref_engine_create(uint32_t layers, uint32_t bpt, uint32_t page_tokens, const char* tag,
                        size_t chunk_size, size_t ram_pool_bytes, size_t store_io_threads,
                        uint32_t num_pages, int layerwise, size_t staging_budget,
                        size_t conn_io_threads, int pin_stores) {
    auto* e = new RefEngine;
    e->scfg.model = make_spec(layers, bpt, page_tokens, tag);
    e->scfg.chunk_size = chunk_size;
    e->scfg.ram_pool_bytes = ram_pool_bytes;
    e->scfg.io_threads = store_io_threads;
    e->store = std::make_unique<TieredStore>(e->scfg);
    e->pages = std::make_unique<PagedKVStore>(e->scfg.model, num_pages);
    Connector::Config c;
    c.mode = layerwise ? TransferMode::layerwise : TransferMode::blocking;
    c.staging_budget_bytes = staging_budget;
    c.io_threads = conn_io_threads;
    c.pin_stores = pin_stores != 0;
    e->conn = std::make_unique<Connector>(*e->store, *e->pages, c);
    return e;
}

void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }

// Pages sized to hold `tokens`, bound per layer (test_connector.cpp:101-113).
int ref_bind_pages(void* h, uint64_t id, size_t tokens) {
    auto* e = static_cast<RefEngine*>(h);
    const auto& sp = e->pages->spec();
    size_t blocks = (tokens + sp.page_tokens - 1) / sp.page_tokens;
    auto alloc = e->pages->alloc_pages(id, blocks * sp.num_layers);
    if (!alloc.ok()) return int(alloc.code());
    for (uint32_t l = 0; l < sp.num_layers; ++l) {
        std::vector<PageId> slice(alloc.value().begin() + size_t(l) * blocks,
                                  alloc.value().begin() + size_t(l + 1) * blocks);
        e->pages->bind_layer(id, l, slice);
    }
    return 0;
}

size_t ref_release_query(void* h, uint64_t id) {
    return static_cast<RefEngine*>(h)->pages->release_query(id).size();
}
size_t ref_free_pages(void* h) { return static_cast<RefEngine*>(h)->pages->free_page_count(); }

// Engine compute stand-in for tokens [from, to) (test_connector.cpp:116-137).
void ref_compute_range(void* h, uint64_t id, const uint32_t* prompt, size_t from, size_t to) {
    auto* e = static_cast<RefEngine*>(h);
    auto& pages = *e->pages;
    const auto& sp = pages.spec();
    uint64_t seed = model_seed_of(sp);
    const size_t pt = sp.page_tokens, bpt = sp.bytes_per_token_per_layer;
    for (uint32_t l = 0; l < sp.num_layers; ++l) {
        auto list = pages.layer_pages(id, l);
        size_t pos = from;
        while (pos < to) {
            size_t page_idx = pos / pt;
            size_t seg = std::min(to, (page_idx + 1) * pt);
            std::vector<uint8_t> buf((seg - pos) * bpt);
            synth_layer_kv(seed, TokenSpanView(prompt + pos, seg - pos), l, pos, uint32_t(bpt),
                           MutByteSpan(buf.data(), buf.size()));
            std::memcpy(pages.page_data(list[page_idx]).data() + (pos - page_idx * pt) * bpt,
                        buf.data(), buf.size());
            pages.mark_populated(list[page_idx], l);
            pos = seg;
        }
    }
}

// gather_tokens over the first ceil(n/pt) pages of one layer.
int ref_gather_layer(void* h, uint64_t id, uint32_t layer, size_t n, uint8_t* out) {
    auto* e = static_cast<RefEngine*>(h);
    const auto& sp = e->pages->spec();
    auto list = e->pages->layer_pages(id, layer);
    list.resize(std::min(list.size(), (n + sp.page_tokens - 1) / sp.page_tokens));
    return int(e->pages->gather_tokens_into(list, layer, n,
                                            MutByteSpan(out, n * sp.bytes_per_token_per_layer))
                   .code);
}

size_t ref_match(void* h, uint64_t id, const uint32_t* prompt, size_t n) {
    return static_cast<RefEngine*>(h)->conn->get_num_new_matched_tokens(id,
                                                                        TokenSpanView(prompt, n));
}

int ref_update_alloc(void* h, uint64_t id, size_t blocks, size_t ext) {
    return int(static_cast<RefEngine*>(h)->conn->update_state_after_alloc(id, blocks, ext).code);
}

// One metadata handle per scheduling iteration; returns its index.
int ref_build_meta(void* h, size_t nq, const uint64_t* ids, const uint32_t* const* prompts,
                   const size_t* lens) {
    auto* e = static_cast<RefEngine*>(h);
    SchedulerOutput out;
    for (size_t i = 0; i < nq; ++i)
        out.queries.push_back({ids[i], std::vector<TokenId>(prompts[i], prompts[i] + lens[i])});
    e->metas.push_back(e->conn->build_connector_meta(out));
    return int(e->metas.size() - 1);
}

int ref_start_load(void* h, int m) {
    auto* e = static_cast<RefEngine*>(h);
    return int(e->conn->start_load_kv(e->metas[m]).code);
}
int ref_wait_load(void* h, int m, uint32_t layer) {
    auto* e = static_cast<RefEngine*>(h);
    return int(e->conn->wait_load_kv(e->metas[m], layer).code);
}
int ref_start_store(void* h, int m) {
    auto* e = static_cast<RefEngine*>(h);
    return int(e->conn->start_store_kv(e->metas[m]).code);
}
int ref_wait_store(void* h, int m, uint32_t layer) {
    auto* e = static_cast<RefEngine*>(h);
    return int(e->conn->wait_store_kv(e->metas[m], layer).code);
}
int ref_meta_layerwise(void* h, int m) {
    return static_cast<RefEngine*>(h)->metas[m].mode() == TransferMode::layerwise;
}
size_t ref_meta_loaded(void* h, int m, uint64_t id) {
    return static_cast<RefEngine*>(h)->metas[m].loaded_tokens(id);
}
void ref_meta_drop(void* h, int m) { static_cast<RefEngine*>(h)->metas[m] = ConnectorMetadata{}; }

// Plan of query `qi` of metadata m. kind 0 = load plan, 1 = store plan. Each
// descriptor is written as 4 u64 (start, end, record_tokens, chunk_index)
// plus 32 digest bytes. Returns the descriptor count; writes at most cap.
size_t ref_meta_plan(void* h, int m, size_t qi, int kind, uint64_t* spans, uint8_t* digests,
                     size_t cap, uint64_t* matched_out) {
    auto* e = static_cast<RefEngine*>(h);
    const auto& plan = e->metas[m].plans().at(qi);
    const auto& v = kind == 0 ? plan.load_plan : plan.store_plan;
    if (matched_out) *matched_out = plan.matched_tokens;
    for (size_t i = 0; i < v.size() && i < cap; ++i) {
        spans[4 * i + 0] = v[i].span.start;
        spans[4 * i + 1] = v[i].span.end;
        spans[4 * i + 2] = v[i].record_tokens;
        spans[4 * i + 3] = v[i].key.chunk_index;
        std::memcpy(digests + 32 * i, v[i].key.digest.data(), 32);
    }
    return v.size();
}

// Per-chunk store statuses of the final wait: codes[i] (Errc), digests[i].
size_t ref_meta_store_results(void* h, int m, uint64_t id, int* codes, uint8_t* digests,
                              size_t cap) {
    auto r = static_cast<RefEngine*>(h)->metas[m].store_results(id);
    for (size_t i = 0; i < r.size() && i < cap; ++i) {
        codes[i] = int(r[i].second.code);
        std::memcpy(digests + 32 * i, r[i].first.digest.data(), 32);
    }
    return r.size();
}

int ref_finish_query(void* h, uint64_t id) {
    auto r = static_cast<RefEngine*>(h)->conn->finish_query(id);
    return int(r.code());
}

// Decode storing (connector.hpp:116-119): the engine hands each generated
// token's per-layer KV to append_decode; here those bytes are the synth KV of
// `token` at absolute position `pos` (what the engine computed).
int ref_begin_decode(void* h, uint64_t id) {
    return int(static_cast<RefEngine*>(h)->conn->begin_decode(id).code);
}
int ref_append_decode(void* h, uint64_t id, uint32_t token, size_t pos) {
    auto* e = static_cast<RefEngine*>(h);
    const auto& sp = e->pages->spec();
    const uint32_t bpt = uint32_t(sp.bytes_per_token_per_layer);
    std::vector<std::vector<uint8_t>> bufs(sp.num_layers, std::vector<uint8_t>(bpt));
    std::vector<ByteSpan> spans;
    for (uint32_t l = 0; l < sp.num_layers; ++l) {
        synth_layer_kv(model_seed_of(sp), TokenSpanView(&token, 1), l, pos, bpt,
                       MutByteSpan(bufs[l].data(), bpt));
        spans.emplace_back(bufs[l].data(), bpt);
    }
    return int(e->conn->append_decode(id, token, spans).code);
}
size_t ref_finish_query_keys(void* h, uint64_t id, uint8_t* digests, size_t cap, int* code) {
    auto r = static_cast<RefEngine*>(h)->conn->finish_query(id);
    *code = int(r.code());
    if (!r.ok()) return 0;
    const auto& keys = r.value();
    for (size_t i = 0; i < keys.size() && i < cap; ++i) std::memcpy(digests + 32 * i, keys[i].digest.data(), 32);
    return keys.size();
}

// --- store (store.hpp:153-171) ----------------------------------------------

int ref_store_contains(void* h, const uint8_t* digest) {
    Digest d;
    std::memcpy(d.data(), digest, 32);
    return !static_cast<RefEngine*>(h)->store->contains(d).empty();
}

// Whole payload of a stored chunk; returns bytes (0 when absent).
size_t ref_store_get(void* h, const uint8_t* digest, uint8_t* out, size_t cap) {
    Digest d;
    std::memcpy(d.data(), digest, 32);
    auto r = static_cast<RefEngine*>(h)->store->get(d);
    if (!r.ok()) return 0;
    auto p = r.value().payload();
    if (out && p.size() <= cap) std::memcpy(out, p.data(), p.size());
    return p.size();
}

size_t ref_store_clear(void* h, const uint8_t* digest) {
    Digest d;
    std::memcpy(d.data(), digest, 32);
    return static_cast<RefEngine*>(h)->store->clear({d}).removed;
}

size_t ref_store_entries(void* h) { return static_cast<RefEngine*>(h)->store->stats().entries; }

// Direct RAM-tier operations (store.hpp:153-171) for the store op-soup
// parity test: put of a caller payload ([L][T][bpt]), pin, get_layer, clear
// with its refused count, and the RAM slot statistics.
int ref_store_put(void* h, const uint8_t* digest, uint32_t token_count, const uint8_t* payload, size_t n,
                  int pin) {
    auto* e = static_cast<RefEngine*>(h);
    const auto& m = e->store->config().model;
    ChunkKey key;
    std::memcpy(key.digest.data(), digest, 32);
    key.model_tag = m.model_tag;
    KVChunkBuilder b(key, token_count, m.num_layers, m.bytes_per_token_per_layer);
    const size_t lb = size_t(token_count) * m.bytes_per_token_per_layer;
    if (n != lb * m.num_layers) return int(Errc::size_mismatch);
    for (uint32_t l = 0; l < m.num_layers; ++l) b.set_layer(l, ByteSpan(payload + l * lb, lb));
    const auto& r = e->store->put(std::move(b).seal(), {TierId::ram()}, pin != 0).wait();
    for (const auto& t : r.tiers)
        if (!t.status.ok()) return int(t.status.code);
    return 0;
}

int ref_store_pin(void* h, const uint8_t* digest, int on) {
    Digest d;
    std::memcpy(d.data(), digest, 32);
    return int(static_cast<RefEngine*>(h)->store->pin(d, TierId::ram(), on != 0).code);
}

int ref_store_get_layer(void* h, const uint8_t* digest, uint32_t layer, uint8_t* out, size_t cap, size_t* n) {
    Digest d;
    std::memcpy(d.data(), digest, 32);
    auto r = static_cast<RefEngine*>(h)->store->get_layer(d, layer);
    *n = 0;
    if (!r.ok()) return int(r.code());
    *n = r.value().size();
    if (out && r.value().size() <= cap) std::memcpy(out, r.value().data(), r.value().size());
    return 0;
}

int ref_store_clear_n(void* h, const uint8_t* digest, size_t* removed, size_t* refused) {
    Digest d;
    std::memcpy(d.data(), digest, 32);
    const auto r = static_cast<RefEngine*>(h)->store->clear({d});
    *removed = r.removed;
    *refused = r.refused;
    return 0;
}

void ref_store_stats(void* h, size_t out[4]) {
    const auto s = static_cast<RefEngine*>(h)->store->stats();
    out[0] = s.entries;
    out[1] = s.ram_slots_total;
    out[2] = s.ram_slots_used;
    out[3] = s.ram_entries;
}

// Store chunk payloads synthesized for prompt[0, n) (test_connector.cpp:71-99).
int ref_seed_store(void* h, const uint32_t* prompt, size_t n) {
    auto* e = static_cast<RefEngine*>(h);
    const auto& cfg = e->store->config();
    TokenSpanView p(prompt, n);
    auto keys = chunk_keys(p, cfg.chunk_size, cfg.model.model_tag);
    auto spans = chunk_tokens(p, cfg.chunk_size);
    uint64_t seed = model_seed_of(cfg.model);
    for (size_t i = 0; i < keys.size(); ++i) {
        KVChunkBuilder b(keys[i], uint32_t(spans[i].length()), cfg.model.num_layers,
                         cfg.model.bytes_per_token_per_layer);
        for (uint32_t l = 0; l < cfg.model.num_layers; ++l)
            synth_layer_kv(seed, p.subspan(spans[i].start, spans[i].length()), l, spans[i].start,
                           cfg.model.bytes_per_token_per_layer, b.layer(l));
        if (!e->store->put(std::move(b).seal(), {TierId::ram()}).wait().all_ok()) return 1;
    }
    return 0;
}

int64_t ref_staging_peak(void* h) { return static_cast<RefEngine*>(h)->conn->staging().peak_bytes(); }
int64_t ref_staging_refs(void* h) {
    return static_cast<RefEngine*>(h)->conn->staging().outstanding_refs();
}

// --- PdStaging (pd_staging.hpp) ----------------------------------------------

void* ref_pd_create() { return new PdStaging; }
void ref_pd_destroy(void* h) { delete static_cast<PdStaging*>(h); }
int ref_pd_register(void* h, uint64_t id) {
    return int(static_cast<PdStaging*>(h)->register_query(id).code);
}
int ref_pd_push(void* h, uint64_t id, uint32_t ordinal, int last, const uint8_t* rec, size_t n) {
    return int(static_cast<PdStaging*>(h)
                   ->push(id, ordinal, last != 0, std::vector<uint8_t>(rec, rec + n))
                   .code);
}
int ref_pd_cancel(void* h, uint64_t id) {
    return int(static_cast<PdStaging*>(h)->cancel(id).code);
}
// Await: concatenated records, first byte of each as a 1-byte tag into tags.
int ref_pd_await(void* h, uint64_t id, uint8_t* tags, size_t cap, size_t* count) {
    auto r = static_cast<PdStaging*>(h)->await(id);
    if (!r.ok()) return int(r.code());
    *count = r.value().size();
    for (size_t i = 0; i < r.value().size() && i < cap; ++i)
        tags[i] = r.value()[i].empty() ? 0 : r.value()[i][0];
    return 0;
}

}  // extern "C"
