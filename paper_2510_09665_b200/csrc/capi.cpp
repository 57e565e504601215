// extern "C" boundary (include/tierkv_b200.h) over the host C++ mirror.
#include "../../include/tierkv_b200.h"

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "connector.hpp"
#include "copy_plan.hpp"
#include "host_copy.hpp"
#include "kernels.hpp"
#include "paged_store.hpp"
#include "pd.hpp"
#include "record.hpp"
#include "store.hpp"
#include "tokens.hpp"

using namespace tkv;

static_assert(sizeof(tkv_paged_layout) == sizeof(PagedLayout));
static_assert(sizeof(tkv_xfer_desc) == sizeof(XferDesc));
static_assert(sizeof(tkv_chain_desc) == sizeof(ChainDesc));
// Device arrays of these cross the ABI by pointer: the field offsets must agree.
static_assert(offsetof(tkv_xfer_desc, layer_stride) == offsetof(XferDesc, layer_stride));
static_assert(offsetof(tkv_xfer_desc, table_dev) == offsetof(XferDesc, table));
static_assert(offsetof(tkv_xfer_desc, first_page) == offsetof(XferDesc, first_page));
static_assert(offsetof(tkv_xfer_desc, n_tokens) == offsetof(XferDesc, n_tokens));
static_assert(offsetof(tkv_chain_desc, n_tokens) == offsetof(ChainDesc, n_tokens));
static_assert(offsetof(tkv_chain_desc, out_first) == offsetof(ChainDesc, out_first));
static_assert(offsetof(tkv_chain_desc, parent) == offsetof(ChainDesc, parent));

// Objects are shared: a connector keeps its store and pages alive, and a
// metadata handle keeps its connector alive, so the C caller may destroy
// handles in any order (each destroy drops one reference).
struct tkv_pages {
    std::shared_ptr<PagedKVStore> p;
    uint64_t shard_offset = 0;  // bytes of the full KV row before this TP shard
};
struct tkv_store {
    std::shared_ptr<TieredStore> s;
};
struct tkv_connector {
    std::shared_ptr<Connector> c;
};
struct tkv_meta {
    std::shared_ptr<Connector> keep;  // destroyed after m (members in reverse order)
    ConnectorMetadata m;
};
struct tkv_pd_staging {
    PdStaging s;
};
struct tkv_pd_sender {
    std::shared_ptr<PagedKVStore> pages;  // kept alive while layers are in flight
    std::unique_ptr<PdLayerSender> s;
};

static_assert(sizeof(tkv_pd_record) == sizeof(PdRecord));
static_assert(sizeof(cudaIpcMemHandle_t) == 64);

namespace {

thread_local std::string g_err;

int fail(Errc c, const std::string& msg) {
    g_err = msg;
    return int(c);
}
int st(const Status& s) {
    if (!s.ok()) g_err = s.to_string();
    return int(s.code);
}

template <typename F>
int guard(F&& f) {
    try {
        return f();
    } catch (const CudaError& e) {
        return fail(Errc::cuda_error, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(Errc::invalid_argument, e.what());
    } catch (const std::exception& e) {
        return fail(Errc::io_error, e.what());
    }
}

int cuda(cudaError_t e) {
    if (e == cudaSuccess) return 0;
    return fail(Errc::cuda_error, cudaGetErrorString(e));
}

ModelSpec to_spec(const tkv_model_spec* s) {
    ModelSpec m;
    m.num_layers = s->num_layers;
    m.bytes_per_token_per_layer = s->bytes_per_token_per_layer;
    m.page_tokens = s->page_tokens;
    m.vocab_size = s->vocab_size ? s->vocab_size : 32000;
    m.model_tag = s->model_tag ? s->model_tag : "";
    return m;
}

Digest to_digest(const uint8_t* p) {
    Digest d;
    std::memcpy(d.data(), p, 32);
    return d;
}

PagedLayout to_layout(const tkv_paged_layout* l) {
    PagedLayout L;
    L.base = l->base;
    L.layer_base = l->layer_base_dev;
    L.page_stride = l->page_stride;
    L.plane_stride = l->plane_stride;
    L.token_stride = l->token_stride;
    L.plane_bytes = l->plane_bytes;
    L.n_planes = l->n_planes;
    L.page_tokens = l->page_tokens;
    L.bpt = l->bpt;
    L.shared_table = l->shared_table;
    return L;
}

std::mutex g_hashers_mu;
std::map<std::pair<std::string, size_t>, std::unique_ptr<KeyHasher>> g_hashers;
KeyHasher& hasher_for(const char* tag, size_t cs) {
    std::lock_guard lock(g_hashers_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    auto key = std::make_pair(std::string(tag) + "#" + std::to_string(dev), cs);
    auto& h = g_hashers[key];
    if (!h) {
        h = std::make_unique<KeyHasher>(tag, cs);
        h->enable_memo(4096);  // repeated prompts through the free functions skip SHA too
    }
    return *h;
}

std::vector<std::vector<TokenId>> to_queries(size_t n, const uint32_t* const* prompts,
                                             const size_t* lens) {
    std::vector<std::vector<TokenId>> v(n);
    for (size_t i = 0; i < n; ++i) v[i].assign(prompts[i], prompts[i] + lens[i]);
    return v;
}

}  // namespace

extern "C" {

const char* tkv_last_error(void) { return g_err.c_str(); }
const char* tkv_errc_name(int code) { return errc_name(Errc(code)); }
const char* tkv_build_info(void) { return "tierkv_b200 sm_100a " __DATE__ " " __TIME__; }
uint64_t tkv_launch_count(void) { return launch_count(); }
void tkv_host_copy(void* dst, const void* src, size_t n) { host_copy(dst, src, n); }

// ---- kernel level -----------------------------------------------------------

int tkv_plan_tiles(const tkv_xfer_desc* descs, uint32_t n, uint32_t page_tokens,
                   uint32_t page_bytes, uint32_t ppt, uint32_t n_layers, uint32_t* tb,
                   uint32_t* ppt_out) {
    if (!page_tokens) return fail(Errc::invalid_argument, "page_tokens == 0");
    if (ppt == 0) ppt = pages_per_tile(page_bytes);
    tb[0] = 0;
    for (uint32_t i = 0; i < n; ++i)
        tb[i + 1] = tb[i] + tiles_for(descs[i].n_tokens, page_tokens, ppt, n_layers);
    if (ppt_out) *ppt_out = ppt;
    return 0;
}

static int paged(const tkv_paged_layout* layout, const tkv_xfer_desc* descs, const uint32_t* tb,
                 uint32_t n_desc, uint32_t tiles, uint32_t l0, uint32_t nl, uint32_t ppt,
                 uint64_t addr_or, int ctas, void* stream, CopyDir dir) {
    PagedCopyPlan P;
    P.descs = reinterpret_cast<const XferDesc*>(descs);
    P.tile_base = tb;
    P.n_desc = n_desc;
    P.total_tiles = tiles;
    P.layer_begin = l0;
    P.n_layers = nl;
    P.pages_per_tile = ppt;
    P.addr_or = addr_or;
    return cuda(launch_paged_copy(to_layout(layout), P, dir, ctas, cudaStream_t(stream)));
}

int tkv_affine_form(const tkv_xfer_desc* descs, uint32_t n, uint32_t page_tokens, tkv_affine_plan* out) {
    if (!descs || !out) return fail(Errc::invalid_argument, "null pointer");
    std::vector<XferDesc> d(reinterpret_cast<const XferDesc*>(descs), reinterpret_cast<const XferDesc*>(descs) + n);
    PagedCopyPlan P;
    if (!affine_form(d, page_tokens, P)) return int(Errc::not_found);
    out->n_desc = n;
    out->pages_per_desc = P.aff_pages;
    out->last_tokens = P.aff_last_tokens;
    out->first_page = P.aff_first_page;
    out->table_dev = P.aff_table;
    out->table_stride = P.aff_table_stride;
    out->pad = 0;
    out->chunk0 = P.aff_chunk0;
    out->chunk_stride = P.aff_chunk_stride;
    out->layer_stride = P.aff_layer_stride;
    return 0;
}

static int paged_affine(const tkv_paged_layout* layout, const tkv_affine_plan* a, uint32_t l0, uint32_t nl,
                        int ctas, void* stream, CopyDir dir) {
    if (!layout || !a) return fail(Errc::invalid_argument, "null pointer");
    if (a->n_desc == 0 || a->pages_per_desc == 0) return fail(Errc::invalid_argument, "empty affine plan");
    PagedCopyPlan P;
    P.n_desc = a->n_desc;
    P.layer_begin = l0;
    P.n_layers = nl;
    P.aff_pages = a->pages_per_desc;
    P.aff_last_tokens = a->last_tokens;
    P.aff_first_page = a->first_page;
    P.aff_table_stride = a->table_stride;
    P.aff_table = a->table_dev;
    P.aff_chunk0 = a->chunk0;
    P.aff_chunk_stride = a->chunk_stride;
    P.aff_layer_stride = a->layer_stride;
    return cuda(launch_paged_copy_affine(to_layout(layout), P, dir, ctas, cudaStream_t(stream)));
}

int tkv_gather_layers_affine(const tkv_paged_layout* layout, const tkv_affine_plan* plan, uint32_t l0,
                             uint32_t nl, int ctas, void* stream) {
    return paged_affine(layout, plan, l0, nl, ctas, stream, CopyDir::gather);
}

int tkv_scatter_layers_affine(const tkv_paged_layout* layout, const tkv_affine_plan* plan, uint32_t l0,
                              uint32_t nl, int ctas, void* stream) {
    return paged_affine(layout, plan, l0, nl, ctas, stream, CopyDir::scatter);
}

int tkv_gather_layers(const tkv_paged_layout* layout, const tkv_xfer_desc* descs, const uint32_t* tb,
                      uint32_t n_desc, uint32_t tiles, uint32_t l0, uint32_t nl, uint32_t ppt,
                      uint64_t addr_or, int ctas, void* stream) {
    return paged(layout, descs, tb, n_desc, tiles, l0, nl, ppt, addr_or, ctas, stream,
                 CopyDir::gather);
}

int tkv_scatter_layers(const tkv_paged_layout* layout, const tkv_xfer_desc* descs,
                       const uint32_t* tb, uint32_t n_desc, uint32_t tiles, uint32_t l0,
                       uint32_t nl, uint32_t ppt, uint64_t addr_or, int ctas, void* stream) {
    return paged(layout, descs, tb, n_desc, tiles, l0, nl, ppt, addr_or, ctas, stream,
                 CopyDir::scatter);
}

int tkv_hash_chains(const uint32_t* tokens, const tkv_chain_desc* chains, uint32_t n_chains,
                    uint32_t chunk_size, const char* tag, uint32_t tag_len, uint8_t* out,
                    void* stream) {
    if (tag_len > uint32_t(kMaxTagBytes)) return fail(Errc::invalid_argument, "tag too long");
    HashParams p;
    p.chunk_size = chunk_size;
    p.tag_len = tag_len;
    std::memcpy(p.tag, tag, tag_len);
    return cuda(launch_hash_chains(tokens, reinterpret_cast<const ChainDesc*>(chains), n_chains, p,
                                   out, cudaStream_t(stream)));
}

int tkv_sm_copy(const void* src, void* dst, uint64_t bytes, void* stream) {
    if (bytes && (!src || !dst)) return fail(Errc::invalid_argument, "null pointer");
    return cuda(launch_sm_copy(src, dst, bytes, cudaStream_t(stream)));
}

int tkv_ce_copy(const void* src, void* dst, uint64_t bytes, void* stream) {
    if (bytes && (!src || !dst)) return fail(Errc::invalid_argument, "null pointer");
    return cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, cudaStream_t(stream)));
}

int tkv_ce_copy_pieces(void* const* dst, const void* const* src, const size_t* sizes, size_t n,
                       int kind, void* stream) {
    if (n && (!dst || !src || !sizes)) return fail(Errc::invalid_argument, "null pointer");
    if (kind != cudaMemcpyHostToDevice && kind != cudaMemcpyDeviceToHost)
        return fail(Errc::invalid_argument, "kind must be 1 (host->device) or 2 (device->host)");
    return cuda(ce_copy_pieces(dst, src, sizes, n, cudaMemcpyKind(kind), cudaStream_t(stream)));
}

size_t tkv_plan_copy_runs(void* const* dst, const void* const* src, const size_t* sizes, size_t n,
                          size_t pitch_max, size_t* first, size_t* rows) {
    std::vector<CopyRun> runs(n);
    const size_t k = plan_copy_runs(dst, src, sizes, n, pitch_max, runs.data());
    for (size_t i = 0; i < k; ++i) {
        if (first) first[i] = runs[i].first;
        if (rows) rows[i] = runs[i].rows;
    }
    return k;
}

static SynthArgs synth_args(const uint32_t* tokens, const int32_t* table, uint32_t stride,
                            uint64_t seed, uint32_t p0, uint32_t p1, uint32_t l0, uint32_t l1) {
    SynthArgs a;
    a.tokens = tokens;
    a.table = table;
    a.table_stride = stride;
    a.seed = seed;
    a.pos_begin = p0;
    a.pos_end = p1;
    a.layer_begin = l0;
    a.layer_end = l1;
    return a;
}

int tkv_synth_pages(const tkv_paged_layout* layout, const uint32_t* tokens, const int32_t* table,
                    uint32_t stride, uint64_t seed, uint32_t p0, uint32_t p1, uint32_t l0,
                    uint32_t l1, void* stream) {
    return cuda(launch_synth_pages(to_layout(layout), synth_args(tokens, table, stride, seed, p0, p1, l0, l1),
                                   cudaStream_t(stream)));
}

int tkv_verify_pages(const tkv_paged_layout* layout, const uint32_t* tokens, const int32_t* table,
                     uint32_t stride, uint64_t seed, uint32_t p0, uint32_t p1, uint32_t l0,
                     uint32_t l1, unsigned long long* mism, void* stream) {
    return cuda(launch_verify_pages(to_layout(layout),
                                    synth_args(tokens, table, stride, seed, p0, p1, l0, l1), mism,
                                    cudaStream_t(stream)));
}

int tkv_synth_chunk(const uint32_t* tokens, uint64_t seed, uint32_t start, uint32_t n,
                    uint32_t n_layers, uint32_t bpt, uint8_t* out, void* stream) {
    return cuda(launch_synth_chunk(tokens, seed, start, n, n_layers, bpt, out, cudaStream_t(stream)));
}

// ---- q8 codec -----------------------------------------------------------------

static_assert(sizeof(tkv_codec_item) == sizeof(CodecItem));

uint64_t tkv_q8_blob_bytes(uint64_t payload) { return q8_blob_bytes(payload); }

int tkv_codec_plan(const tkv_codec_item* items, uint32_t n, uint32_t* seg_base) {
    seg_base[0] = 0;
    for (uint32_t i = 0; i < n; ++i) seg_base[i + 1] = seg_base[i] + codec_segments(items[i].bytes);
    return 0;
}

uint64_t tkv_q8_encode_scratch_bytes(uint32_t n) { return q8_encode_scratch_bytes(n); }

int tkv_q8_encode(const tkv_codec_item* items, const uint32_t* seg_base, uint32_t n, uint32_t segs,
                  int* maxabs, void* stream) {
    return cuda(launch_q8_encode(reinterpret_cast<const CodecItem*>(items), seg_base, n, segs, maxabs,
                                 cudaStream_t(stream)));
}

int tkv_q8_decode(const tkv_codec_item* items, const uint32_t* seg_base, uint32_t n, uint32_t segs,
                  void* stream) {
    return cuda(launch_q8_decode(reinterpret_cast<const CodecItem*>(items), seg_base, n, segs,
                                 cudaStream_t(stream)));
}

// ---- keys -------------------------------------------------------------------

int tkv_chunk_keys(const char* tag, size_t cs, const uint32_t* tokens, size_t n, uint8_t* out,
                   size_t* n_chunks) {
    return guard([&] {
        auto keys = chunk_keys(hasher_for(tag, cs), TokenSpanView(tokens, n));
        for (size_t i = 0; i < keys.size(); ++i) std::memcpy(out + 32 * i, keys[i].digest.data(), 32);
        *n_chunks = keys.size();
        return 0;
    });
}

int tkv_keychain_next(const char* tag, size_t cs, const uint8_t* parent, const uint32_t* tokens,
                      size_t n, uint8_t* out) {
    return guard([&] {
        KeyChain chain(hasher_for(tag, cs));
        chain.reset(to_digest(parent), 0);
        auto k = chain.next(TokenSpanView(tokens, n));
        std::memcpy(out, k.digest.data(), 32);
        return 0;
    });
}

// ---- pages ------------------------------------------------------------------

int tkv_pages_create(const tkv_model_spec* spec, uint32_t num_pages, int device, tkv_pages** out) {
    return guard([&] {
        if (device >= 0) TKV_CUDA(cudaSetDevice(device));
        auto* p = new tkv_pages;
        p->p = std::make_shared<PagedKVStore>(to_spec(spec), num_pages, device);
        *out = p;
        return 0;
    });
}
void tkv_pages_destroy(tkv_pages* p) {
    if (p) cudaDeviceSynchronize();
    delete p;
}
int tkv_pages_alloc(tkv_pages* p, uint64_t q, size_t n, uint32_t* ids) {
    return guard([&] {
        auto r = p->p->alloc_pages(q, n);
        if (!r.ok()) return st(r.status());
        std::memcpy(ids, r.value().data(), n * sizeof(uint32_t));
        return 0;
    });
}
int tkv_pages_bind_layer(tkv_pages* p, uint64_t q, uint32_t layer, const uint32_t* ids, size_t n) {
    return guard([&] {
        p->p->bind_layer(q, layer, std::vector<PageId>(ids, ids + n));
        return 0;
    });
}
int tkv_pages_admit(tkv_pages* p, uint64_t q, size_t tokens) {
    return guard([&] { return st(p->p->admit(q, tokens)); });
}
size_t tkv_pages_layer_pages(tkv_pages* p, uint64_t q, uint32_t layer, uint32_t* ids, size_t cap) {
    auto v = p->p->layer_pages(q, layer);
    if (ids) std::memcpy(ids, v.data(), std::min(cap, v.size()) * sizeof(uint32_t));
    return v.size();
}
size_t tkv_pages_release(tkv_pages* p, uint64_t q) { return p->p->release_query(q).size(); }
size_t tkv_pages_free_count(tkv_pages* p) { return p->p->free_page_count(); }
size_t tkv_pages_allocated_count(tkv_pages* p) { return p->p->allocated_page_count(); }
size_t tkv_pages_pool_pages(tkv_pages* p) { return p->p->pool_pages(); }
int tkv_pages_mark_populated(tkv_pages* p, uint32_t page, uint32_t layer) {
    if (page >= p->p->pool_pages()) return fail(Errc::invalid_argument, "page id out of range");
    p->p->mark_populated(page, layer);
    return 0;
}
int tkv_pages_populated(tkv_pages* p, uint32_t page) {
    return page < p->p->pool_pages() && p->p->populated(page);
}
int tkv_pages_gather(tkv_pages* p, const uint32_t* ids, size_t n_ids, uint32_t layer, size_t tokens,
                     uint8_t* out, size_t out_bytes) {
    return guard([&] {
        TKV_CUDA(cudaDeviceSynchronize());
        return st(p->p->gather_tokens_into(std::vector<PageId>(ids, ids + n_ids), layer, tokens, out,
                                           out_bytes));
    });
}
int tkv_pages_scatter(tkv_pages* p, const uint8_t* buf, size_t bytes, const uint32_t* ids,
                      size_t n_ids, uint32_t layer, size_t tokens) {
    return guard([&] {
        TKV_CUDA(cudaDeviceSynchronize());
        return st(p->p->scatter_tokens(buf, bytes, std::vector<PageId>(ids, ids + n_ids), layer, tokens));
    });
}
int tkv_pages_layout(tkv_pages* p, tkv_paged_layout* out) {
    const PagedLayout L = p->p->layout();
    out->base = L.base;
    out->layer_base_dev = L.layer_base;
    out->page_stride = L.page_stride;
    out->plane_stride = L.plane_stride;
    out->token_stride = L.token_stride;
    out->plane_bytes = L.plane_bytes;
    out->n_planes = L.n_planes;
    out->page_tokens = L.page_tokens;
    out->bpt = L.bpt;
    out->shared_table = L.shared_table;
    return 0;
}
int tkv_pages_device_table(tkv_pages* p, uint64_t q, void* stream, const int32_t** table,
                           uint32_t* stride) {
    return guard([&] {
        auto t = p->p->device_table(q, cudaStream_t(stream));
        if (!t.ok()) return st(t.status());
        *table = t.value().ptr;
        *stride = t.value().stride;
        return 0;
    });
}

static int pages_synth(tkv_pages* p, uint64_t q, const uint32_t* tokens, uint32_t from, uint32_t to,
                       uint32_t l0, uint32_t l1, unsigned long long* mism, void* stream) {
    return guard([&] {
        const auto& sp = p->p->spec();
        if (l1 > sp.num_layers || l0 > l1 || from > to)
            return fail(Errc::invalid_argument, "range");
        for (uint32_t l = l0; l < l1; ++l) {
            const size_t have = p->p->layer_pages(q, l).size() * sp.page_tokens;
            if (to > have) return fail(Errc::size_mismatch, "positions beyond the query's pages");
        }
        auto t = p->p->device_table(q, cudaStream_t(stream));
        if (!t.ok()) return st(t.status());
        SynthArgs a = synth_args(tokens, t.value().ptr, t.value().stride, sp.model_seed(), from, to, l0, l1);
        a.row_offset = p->shard_offset;
        if (mism) return cuda(launch_verify_pages(p->p->layout(), a, mism, cudaStream_t(stream)));
        int rc = cuda(launch_synth_pages(p->p->layout(), a, cudaStream_t(stream)));
        if (rc) return rc;
        if (to > from) {
            const uint32_t pt = sp.page_tokens;
            for (uint32_t l = l0; l < l1; ++l) {
                auto list = p->p->layer_pages(q, l);
                for (uint32_t pg = from / pt; pg <= (to - 1) / pt; ++pg) p->p->mark_populated(list[pg], l);
            }
        }
        return 0;
    });
}

int tkv_pages_set_shard(tkv_pages* p, uint64_t byte_offset) {
    if (byte_offset % 8) return fail(Errc::invalid_argument, "shard offset must be a multiple of 8");
    p->shard_offset = byte_offset;
    return 0;
}
int tkv_pages_compute(tkv_pages* p, uint64_t q, const uint32_t* tokens, uint32_t from, uint32_t to,
                      uint32_t l0, uint32_t l1, void* stream) {
    return pages_synth(p, q, tokens, from, to, l0, l1, nullptr, stream);
}
int tkv_pages_verify(tkv_pages* p, uint64_t q, const uint32_t* tokens, uint32_t from, uint32_t to,
                     uint32_t l0, uint32_t l1, unsigned long long* mism, void* stream) {
    if (!mism) return fail(Errc::invalid_argument, "null mismatch counter");
    return pages_synth(p, q, tokens, from, to, l0, l1, mism, stream);
}

// ---- store ------------------------------------------------------------------

int tkv_store_create(const tkv_model_spec* spec, size_t chunk_size, size_t ram_bytes, tkv_store** out) {
    return guard([&] {
        StoreConfig cfg;
        cfg.model = to_spec(spec);
        cfg.chunk_size = chunk_size;
        cfg.ram_pool_bytes = ram_bytes;
        auto* s = new tkv_store;
        s->s = std::make_shared<TieredStore>(cfg);
        *out = s;
        return 0;
    });
}
void tkv_store_destroy(tkv_store* s) { delete s; }
int tkv_store_verify_synth(tkv_store* s, const uint8_t* digest, const uint32_t* tokens_dev, uint64_t seed,
                           uint32_t start, uint64_t row_offset, unsigned long long* mismatches_dev,
                           void* stream) {
    return guard([&] {
        Digest d;
        std::memcpy(d.data(), digest, 32);
        auto r = s->s->acquire(d, 0);
        if (!r.ok()) return st(r.status());
        const auto& m = s->s->config().model;
        cudaError_t e = launch_verify_chunk(tokens_dev, seed, start, r.value().token_count, m.num_layers,
                                            uint32_t(m.bytes_per_token_per_layer), row_offset, r.value().dev,
                                            mismatches_dev, cudaStream_t(stream));
        if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStream_t(stream));
        s->s->release(d);
        return cuda(e);
    });
}
int tkv_store_put(tkv_store* s, const uint8_t* digest, uint32_t tokens, const uint8_t* payload,
                  size_t bytes, int pin) {
    return guard([&] { return st(s->s->put(to_digest(digest), tokens, payload, bytes, pin != 0).wait()); });
}
int tkv_store_get(tkv_store* s, const uint8_t* digest, uint8_t* out, size_t cap, size_t* n) {
    return guard([&] {
        auto r = s->s->get(to_digest(digest));
        if (!r.ok()) return st(r.status());
        *n = r.value().size();
        if (out && r.value().size() <= cap) std::memcpy(out, r.value().data(), r.value().size());
        return 0;
    });
}
int tkv_store_get_layer(tkv_store* s, const uint8_t* digest, uint32_t layer, uint8_t* out,
                        size_t cap, size_t* n) {
    return guard([&] {
        auto r = s->s->get_layer(to_digest(digest), layer);
        if (!r.ok()) return st(r.status());
        *n = r.value().size();
        if (out && r.value().size() <= cap) std::memcpy(out, r.value().data(), r.value().size());
        return 0;
    });
}
int tkv_store_contains(tkv_store* s, const uint8_t* digest) { return s->s->contains(to_digest(digest)); }
int tkv_store_pin(tkv_store* s, const uint8_t* digest, int on) {
    return st(s->s->pin(to_digest(digest), on != 0));
}
int tkv_store_clear(tkv_store* s, const uint8_t* digests, size_t n, size_t* removed, size_t* refused) {
    std::vector<Digest> v(n);
    for (size_t i = 0; i < n; ++i) v[i] = to_digest(digests + 32 * i);
    auto r = s->s->clear(v);
    if (removed) *removed = r.removed;
    if (refused) *refused = r.refused;
    return 0;
}
int tkv_store_stats(tkv_store* s, size_t out[4]) {
    auto r = s->s->stats();
    out[0] = r.entries;
    out[1] = r.ram_slots_total;
    out[2] = r.ram_slots_used;
    out[3] = r.ram_entries;
    return 0;
}

int tkv_model_tag_hash(const char* tag, uint64_t* out) {
    return guard([&] {
        const size_t n = std::strlen(tag);
        PinnedBuffer buf(n + 32 + 16);
        std::memcpy(buf.host, tag, n);
        TKV_CUDA(launch_sha256_bytes(buf.dev, uint32_t(n), buf.dev + ((n + 15) & ~size_t(15)), nullptr));
        TKV_CUDA(cudaStreamSynchronize(nullptr));
        const uint8_t* d = buf.host + ((n + 15) & ~size_t(15));
        uint64_t v = 0;
        for (int i = 7; i >= 0; --i) v = (v << 8) | d[i];
        *out = v;
        return 0;
    });
}
int tkv_store_export_record(tkv_store* s, const uint8_t* digest, uint64_t tag_hash, uint8_t* out,
                            size_t cap, size_t* n) {
    return guard([&] {
        return st(s->s->export_record_into(to_digest(digest), tag_hash, out, cap, n));
    });
}
int tkv_store_import_record(tkv_store* s, const uint8_t* record, size_t n, int pin) {
    return guard([&] { return st(s->s->import_record(record, n, pin != 0)); });
}
int tkv_record_peek(const uint8_t* record, size_t n, uint8_t* digest, uint32_t* geo, uint64_t* tag_hash) {
    auto r = peek_record(record, n);
    if (!r.ok()) return st(r.status());
    std::memcpy(digest, r.value().digest.data(), 32);
    geo[0] = r.value().token_count;
    geo[1] = r.value().num_layers;
    geo[2] = r.value().bytes_per_token;
    *tag_hash = r.value().model_tag_hash;
    return 0;
}

// ---- connector --------------------------------------------------------------

void tkv_connector_config_default(tkv_connector_config* cfg) {
    Connector::Config d;
    cfg->layerwise = d.mode == TransferMode::layerwise;
    cfg->pin_stores = d.pin_stores;
    cfg->staging_budget_bytes = d.staging_budget_bytes;
    cfg->staging_depth = d.staging_depth;
    cfg->load_zero_copy = d.load_path == LoadPath::zero_copy;
    cfg->store_zero_copy = d.store_path == StorePath::zero_copy;
    cfg->store_ctas = d.store_ctas;
    cfg->load_ctas = d.load_ctas;
    cfg->engine_stream = d.engine_stream;
    cfg->memo_entries = d.memo_entries;
}

int tkv_connector_create(tkv_store* s, tkv_pages* p, const tkv_connector_config* cfg,
                         tkv_connector** out) {
    return guard([&] {
        Connector::Config c;
        if (cfg) {
            c.mode = cfg->layerwise ? TransferMode::layerwise : TransferMode::blocking;
            c.pin_stores = cfg->pin_stores != 0;
            c.staging_budget_bytes = cfg->staging_budget_bytes;
            c.staging_depth = cfg->staging_depth;
            c.load_path = cfg->load_zero_copy ? LoadPath::zero_copy : LoadPath::copy_engine;
            c.store_path = cfg->store_zero_copy ? StorePath::zero_copy : StorePath::copy_engine;
            c.store_ctas = cfg->store_ctas > 0 ? cfg->store_ctas : c.store_ctas;
            c.load_ctas = cfg->load_ctas;
            c.engine_stream = cudaStream_t(cfg->engine_stream);
            c.memo_entries = cfg->memo_entries;
        }
        auto* h = new tkv_connector;
        // the deleter's captures release the store and pages after the connector
        std::shared_ptr<TieredStore> store = s->s;
        std::shared_ptr<PagedKVStore> pages = p->p;
        h->c = std::shared_ptr<Connector>(new Connector(*store, *pages, c),
                                          [store, pages](Connector* x) { delete x; });
        *out = h;
        return 0;
    });
}
void tkv_connector_destroy(tkv_connector* c) { delete c; }

int tkv_connector_get_num_new_matched_tokens(tkv_connector* c, uint64_t q, const uint32_t* tokens,
                                             size_t n, size_t* matched) {
    return guard([&] {
        *matched = c->c->get_num_new_matched_tokens(q, TokenSpanView(tokens, n));
        return 0;
    });
}
int tkv_connector_lookup_batch(tkv_connector* c, size_t nq, const uint64_t* ids,
                               const uint32_t* const* prompts, const size_t* lens, size_t* matched) {
    return guard([&] {
        std::vector<QueryId> q(ids, ids + nq);
        std::vector<TokenSpanView> v(nq);
        for (size_t i = 0; i < nq; ++i) v[i] = TokenSpanView(prompts[i], lens[i]);
        auto r = c->c->get_num_new_matched_tokens(q, v);
        std::memcpy(matched, r.data(), nq * sizeof(size_t));
        return 0;
    });
}
int tkv_connector_update_state_after_alloc(tkv_connector* c, uint64_t q, size_t blocks, size_t ext) {
    return guard([&] { return st(c->c->update_state_after_alloc(q, blocks, ext)); });
}
int tkv_connector_build_meta(tkv_connector* c, size_t nq, const uint64_t* ids,
                             const uint32_t* const* prompts, const size_t* lens, tkv_meta** out) {
    return guard([&] {
        SchedulerOutput so;
        auto qs = to_queries(nq, prompts, lens);
        for (size_t i = 0; i < nq; ++i) so.queries.push_back({ids[i], std::move(qs[i])});
        auto* m = new tkv_meta;
        m->keep = c->c;
        m->m = c->c->build_connector_meta(so);
        *out = m;
        return 0;
    });
}
int tkv_connector_start_load_kv(tkv_connector* c, tkv_meta* m) {
    return guard([&] { return st(c->c->start_load_kv(m->m)); });
}
int tkv_connector_wait_load_kv(tkv_connector* c, tkv_meta* m, uint32_t layer) {
    return guard([&] { return st(c->c->wait_load_kv(m->m, layer)); });
}
int tkv_connector_start_store_kv(tkv_connector* c, tkv_meta* m) {
    return guard([&] { return st(c->c->start_store_kv(m->m)); });
}
int tkv_connector_wait_store_kv(tkv_connector* c, tkv_meta* m, uint32_t layer) {
    return guard([&] { return st(c->c->wait_store_kv(m->m, layer)); });
}
int tkv_connector_prefetch(tkv_connector* c, const uint32_t* tokens, size_t n) {
    return guard([&] {
        c->c->prefetch(TokenSpanView(tokens, n));
        return 0;
    });
}
int tkv_connector_drain_prefetch(tkv_connector* c) {
    return guard([&] {
        c->c->drain_prefetch();
        return 0;
    });
}
int tkv_connector_begin_decode(tkv_connector* c, uint64_t q) {
    return guard([&] { return st(c->c->begin_decode(q)); });
}
int tkv_connector_append_decode(tkv_connector* c, uint64_t q, uint32_t token) {
    return guard([&] { return st(c->c->append_decode(q, token)); });
}
int tkv_connector_append_decode_batch(tkv_connector* c, size_t n, const uint64_t* queries,
                                      const uint32_t* tokens, int* statuses) {
    return guard([&] {
        std::vector<Status> st_(n);
        c->c->append_decode_batch(queries, tokens, n, st_.data());
        for (size_t i = 0; i < n; ++i) statuses[i] = int(st_[i].code);
        return 0;
    });
}
int tkv_connector_finish_query(tkv_connector* c, uint64_t q, uint8_t* out, size_t cap, size_t* n) {
    return guard([&] {
        auto r = c->c->finish_query(q);
        if (!r.ok()) return st(r.status());
        *n = r.value().size();
        for (size_t i = 0; i < r.value().size() && i < cap; ++i)
            std::memcpy(out + 32 * i, r.value()[i].digest.data(), 32);
        return 0;
    });
}
size_t tkv_connector_staging_peak(tkv_connector* c) { return c->c->staging_peak_bytes(); }
void tkv_connector_copy_runs(tkv_connector* c, uint64_t out[2]) {
    const auto s = c->c->copy_stats();
    out[0] = s.pieces;
    out[1] = s.runs;
}
int tkv_connector_memo_stats(tkv_connector* c, uint64_t out[5]) {
    return guard([&] {
        auto s = c->c->hasher().memo_stats();
        out[0] = s.hits;
        out[1] = s.misses;
        out[2] = s.capacity;
        out[3] = s.resets;
        out[4] = s.rehashes;
        return 0;
    });
}
int tkv_connector_debug_poison_memo(tkv_connector* c) {
    return guard([&] {
        c->c->hasher().debug_poison_memo();
        return 0;
    });
}
uint64_t tkv_connector_hash_launches(tkv_connector* c) { return c->c->hasher().launches(); }
uint64_t tkv_connector_lookups_host_decided(tkv_connector* c) { return c->c->hasher().host_decided(); }
uint64_t tkv_connector_lookups_witnessed(tkv_connector* c) {
    try {
        return c->c->hasher().memo_stats().witnessed;
    } catch (...) {
        return 0;
    }
}

// ---- PD -----------------------------------------------------------------------

int tkv_pd_staging_create(tkv_pd_staging** out) {
    return guard([&] {
        *out = new tkv_pd_staging;
        return 0;
    });
}
void tkv_pd_staging_destroy(tkv_pd_staging* s) { delete s; }
int tkv_pd_register(tkv_pd_staging* s, uint64_t q) { return st(s->s.register_query(q)); }
int tkv_pd_push(tkv_pd_staging* s, uint64_t q, uint32_t ordinal, int last, const tkv_pd_record* rec) {
    PdRecord r{rec->addr, rec->bytes, rec->token_count, rec->first_token};
    return st(s->s.push(q, ordinal, last != 0, r));
}
int tkv_pd_await(tkv_pd_staging* s, uint64_t q, tkv_pd_record* out, size_t cap, size_t* n) {
    return guard([&] {
        auto r = s->s.await(q);
        if (!r.ok()) return st(r.status());
        *n = r.value().size();
        for (size_t i = 0; i < r.value().size() && i < cap; ++i) {
            const auto& x = r.value()[i];
            out[i] = tkv_pd_record{x.addr, x.bytes, x.token_count, x.first_token};
        }
        return 0;
    });
}
int tkv_pd_cancel(tkv_pd_staging* s, uint64_t q) { return st(s->s.cancel(q)); }
size_t tkv_pd_registered(tkv_pd_staging* s) { return s->s.registered(); }
int tkv_pd_send(tkv_pages* src, uint64_t q, size_t n_tokens, size_t chunk_size, uint64_t landing,
                uint64_t stride, void* stream, tkv_pd_record* out, size_t cap, size_t* n) {
    return guard([&] {
        auto r = pd_send_chunks(*src->p, q, n_tokens, chunk_size, landing, stride, cudaStream_t(stream));
        if (!r.ok()) return st(r.status());
        *n = r.value().size();
        for (size_t i = 0; i < r.value().size() && i < cap; ++i) {
            const auto& x = r.value()[i];
            out[i] = tkv_pd_record{x.addr, x.bytes, x.token_count, x.first_token};
        }
        return 0;
    });
}
int tkv_pd_sender_begin(tkv_pages* src, uint64_t q, size_t n_tokens, size_t unit_tokens, uint64_t landing,
                        uint64_t unit_stride, tkv_pd_sender** out) {
    return guard([&] {
        auto h = std::make_unique<tkv_pd_sender>();
        h->pages = src->p;
        h->s = std::make_unique<PdLayerSender>(*src->p, q, n_tokens, unit_tokens, landing, unit_stride);
        if (!h->s->status().ok()) return st(h->s->status());
        *out = h.release();
        return 0;
    });
}
int tkv_pd_sender_layer(tkv_pd_sender* s, uint32_t layer, void* engine_stream) {
    return guard([&] { return st(s->s->send_layer(layer, cudaStream_t(engine_stream))); });
}
int tkv_pd_sender_finish(tkv_pd_sender* s, tkv_pd_record* out, size_t cap, size_t* n) {
    return guard([&] {
        auto r = s->s->finish();
        if (!r.ok()) return st(r.status());
        *n = r.value().size();
        for (size_t i = 0; i < r.value().size() && i < cap; ++i) {
            const auto& x = r.value()[i];
            out[i] = tkv_pd_record{x.addr, x.bytes, x.token_count, x.first_token};
        }
        return 0;
    });
}
void tkv_pd_sender_destroy(tkv_pd_sender* s) { delete s; }

int tkv_pd_send_staged(tkv_pages* src, uint64_t q, size_t n_tokens, size_t chunk_size, uint64_t landing,
                       uint64_t stride, uint64_t staging, uint64_t group_bytes, void* stream,
                       tkv_pd_record* out, size_t cap, size_t* n) {
    return guard([&] {
        if (!staging) return fail(Errc::invalid_argument, "null staging buffer");
        auto r = pd_send_chunks_staged(*src->p, q, n_tokens, chunk_size, landing, stride, staging,
                                       cudaStream_t(stream), group_bytes ? group_bytes : (1ull << 30));
        if (!r.ok()) return st(r.status());
        *n = r.value().size();
        for (size_t i = 0; i < r.value().size() && i < cap; ++i) {
            const auto& x = r.value()[i];
            out[i] = tkv_pd_record{x.addr, x.bytes, x.token_count, x.first_token};
        }
        return 0;
    });
}
int tkv_pd_land(tkv_pages* dst, uint64_t q, const tkv_pd_record* recs, size_t n, void* stream) {
    return guard([&] {
        std::vector<PdRecord> v(n);
        for (size_t i = 0; i < n; ++i)
            v[i] = PdRecord{recs[i].addr, recs[i].bytes, recs[i].token_count, recs[i].first_token};
        return st(pd_land_chunks(*dst->p, q, v, cudaStream_t(stream)));
    });
}
int tkv_enable_peer_access(int device, int peer) {
    return guard([&] { return st(enable_peer_access(device, peer)); });
}
// An IPC handle names the whole cudaMalloc allocation and maps at its base,
// so a buffer carved out of a larger allocation (a caching allocator's
// segment) travels as handle + offset from the allocation base. The base
// comes from the driver's cuMemGetAddressRange, reached through the runtime
// (no link-time libcuda dependency).
int tkv_ipc_get_handle(void* ptr, uint8_t* handle64, uint64_t* offset) {
    using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
    static GetRange get_range = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess)
            fn = nullptr;
        return reinterpret_cast<GetRange>(fn);
    }();
    cudaIpcMemHandle_t h;
    int rc = cuda(cudaIpcGetMemHandle(&h, ptr));
    if (rc != 0) return rc;
    unsigned long long base = 0;
    size_t size = 0;
    if (!get_range || get_range(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0)
        return fail(Errc::cuda_error, "cuMemGetAddressRange failed");
    std::memcpy(handle64, &h, sizeof h);
    *offset = reinterpret_cast<unsigned long long>(ptr) - base;
    return 0;
}
int tkv_ipc_open_handle(const uint8_t* handle64, uint64_t offset, void** out) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    void* base = nullptr;
    int rc = cuda(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    if (rc == 0) *out = static_cast<uint8_t*>(base) + offset;
    return rc;
}
int tkv_ipc_close(void* ptr, uint64_t offset) {
    return cuda(cudaIpcCloseMemHandle(static_cast<uint8_t*>(ptr) - offset));
}

int tkv_meta_timeline(tkv_meta* m, float* out, size_t cap, size_t* n) {
    return guard([&] {
        auto t = m->m.timeline();
        *n = t.size();
        std::memcpy(out, t.data(), std::min(cap, t.size()) * sizeof(float));
        return 0;
    });
}

int tkv_meta_origin_since(tkv_meta* m, void* ev, float* ms) {
    return guard([&] {
        *ms = m->m.origin_since(cudaEvent_t(ev));
        return 0;
    });
}

void tkv_meta_destroy(tkv_meta* m) { delete m; }
int tkv_meta_layerwise(tkv_meta* m) { return m->m.mode() == TransferMode::layerwise; }
size_t tkv_meta_loaded_tokens(tkv_meta* m, uint64_t q) { return m->m.loaded_tokens(q); }
size_t tkv_meta_num_plans(tkv_meta* m) { return m->m.plans().size(); }
int tkv_meta_plan(tkv_meta* m, size_t qi, int kind, uint64_t* spans, uint8_t* digests, size_t cap,
                  size_t* n, uint64_t* matched) {
    const auto& plans = m->m.plans();
    if (qi >= plans.size()) return fail(Errc::invalid_argument, "plan index");
    const auto& v = kind == 0 ? plans[qi].load_plan : plans[qi].store_plan;
    if (matched) *matched = plans[qi].matched_tokens;
    *n = v.size();
    for (size_t i = 0; i < v.size() && i < cap; ++i) {
        spans[4 * i] = v[i].span.start;
        spans[4 * i + 1] = v[i].span.end;
        spans[4 * i + 2] = v[i].record_tokens;
        spans[4 * i + 3] = v[i].key.chunk_index;
        std::memcpy(digests + 32 * i, v[i].key.digest.data(), 32);
    }
    return 0;
}
int tkv_meta_store_results(tkv_meta* m, uint64_t q, int* codes, uint8_t* digests, size_t cap,
                           size_t* n) {
    auto r = m->m.store_results(q);
    *n = r.size();
    for (size_t i = 0; i < r.size() && i < cap; ++i) {
        codes[i] = int(r[i].second.code);
        std::memcpy(digests + 32 * i, r[i].first.digest.data(), 32);
    }
    return 0;
}

}  // extern "C"
