/* tierkv_b200 — C-ABI of the B200 KV-cache data-movement path.
 *
 * Drop-in boundary for the reference tierkv hot path (arXiv 2510.09665,
 * /root/reference/proj). Every entry point is extern "C", takes plain
 * pointers and sizes, and returns an int status whose values are the
 * reference's Errc (include/tierkv/common.hpp:13-31) plus TKV_CUDA_ERROR.
 * Device pointers are marked _dev; `stream` is a cudaStream_t passed as
 * void*. tkv_last_error() returns the detail string of the calling thread's
 * last failure.
 *
 * Two layers:
 *  1. kernel level (stream-ordered, no host sync, no allocation):
 *     tkv_gather_layers / tkv_scatter_layers (K1/K2), tkv_hash_chains (K3),
 *     tkv_synth_pages / tkv_verify_pages / tkv_synth_chunk (K4);
 *  2. object level, mirroring the reference C++ classes the engine binds:
 *     tkv_pages_* (PagedKVStore), tkv_store_* (TieredStore RAM tier),
 *     tkv_connector_* + tkv_meta_* (Connector + ConnectorMetadata),
 *     tkv_pd_* (PdStaging + NVLink/P2P chunk sends).
 */
#ifndef TIERKV_B200_H
#define TIERKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: include/tierkv/common.hpp:13-31 ----------------------- */
enum {
    TKV_OK = 0,
    TKV_NOT_FOUND,
    TKV_TIER_FULL,
    TKV_OUT_OF_PAGES,
    TKV_DUPLICATE_KEY,
    TKV_CORRUPT_CHUNK,
    TKV_SIZE_MISMATCH,
    TKV_UNPOPULATED_PAGE,
    TKV_UNKNOWN_CODEC,
    TKV_UNKNOWN_INSTANCE,
    TKV_UNKNOWN_QUERY,
    TKV_INCONSISTENT_ALLOC,
    TKV_CHUNK_MISSING,
    TKV_PINNED,
    TKV_PROTOCOL_ERROR,
    TKV_IO_ERROR,
    TKV_INVALID_ARGUMENT,
    TKV_CUDA_ERROR /* device failure; no reference equivalent */
};

const char* tkv_last_error(void);
const char* tkv_errc_name(int code);
/* Library version / build id of the loaded kernels. */
const char* tkv_build_info(void);
/* Kernel launches issued by this library since load (bench gpu_launches). */
uint64_t tkv_launch_count(void);
/* The connector's host copy of prompt-sized buffers (memcpy semantics; split
 * over helper threads with streaming stores from 128 KiB on). Exported for
 * tests. */
void tkv_host_copy(void* dst, const void* src, size_t n);

/* ---- geometry: include/tierkv/model.hpp:11-33 ----------------------------- */
typedef struct tkv_model_spec {
    uint32_t num_layers;
    uint32_t bytes_per_token_per_layer;
    uint32_t page_tokens;
    uint32_t vocab_size;
    const char* model_tag;
} tkv_model_spec;

/* ========================================================================== *
 * 1. Kernel level
 * ========================================================================== */

/* Paged side of K1/K2. Reference layout (paged_store.hpp:19-82): n_planes=1,
 * token_stride=plane_bytes=bpt, page_stride=page_tokens*bpt, per-layer page
 * lists. vLLM layout: n_planes=2 (K,V), plane_bytes=H*D*elt, per-layer bases
 * in layer_base_dev, shared_table=1 (one block table for all layers). */
typedef struct tkv_paged_layout {
    uint64_t base;
    const uint64_t* layer_base_dev;
    uint64_t page_stride;
    uint64_t plane_stride;
    uint32_t token_stride;
    uint32_t plane_bytes;
    uint32_t n_planes;
    uint32_t page_tokens;
    uint32_t bpt;
    uint32_t shared_table;
} tkv_paged_layout;

/* One chunk transfer (ChunkDescriptor, connector.hpp:22-27): rows
 * [first_page*page_tokens, +n_tokens) of every moved layer, chunk side at
 * chunk + layer*layer_stride + row*bpt (HBM, mapped pinned host or peer). */
typedef struct tkv_xfer_desc {
    uint64_t chunk;
    uint64_t layer_stride;
    const int32_t* table_dev; /* [layers][table_stride] page ids */
    uint32_t table_stride;
    uint32_t first_page;
    uint32_t n_tokens;
    uint32_t pad;
} tkv_xfer_desc;

/* Host helper: tile prefix (n+1 entries) for a launch over n_layers layers.
 * pages_per_tile = 0 picks the default (about 64 KiB per tile). Returns the
 * pages_per_tile used through *ppt_out. */
int tkv_plan_tiles(const tkv_xfer_desc* descs, uint32_t n, uint32_t page_tokens,
                   uint32_t page_bytes, uint32_t pages_per_tile, uint32_t n_layers,
                   uint32_t* tile_base_out, uint32_t* ppt_out);

/* K1: pages -> chunk buffers. Replaces PagedKVStore::gather_tokens_into
 * (src/paged_store.cpp:123-140) for every (chunk, layer) of a batch in one
 * launch. addr_or = OR of all desc.chunk and desc.layer_stride (alignment). */
int tkv_gather_layers(const tkv_paged_layout* layout, const tkv_xfer_desc* descs_dev,
                      const uint32_t* tile_base_dev, uint32_t n_desc, uint32_t total_tiles,
                      uint32_t layer_begin, uint32_t n_layers, uint32_t pages_per_tile,
                      uint64_t addr_or, int ctas, void* stream);
/* K2: chunk buffers -> pages. Replaces PagedKVStore::scatter_tokens
 * (src/paged_store.cpp:147-175). */
int tkv_scatter_layers(const tkv_paged_layout* layout, const tkv_xfer_desc* descs_dev,
                       const uint32_t* tile_base_dev, uint32_t n_desc, uint32_t total_tiles,
                       uint32_t layer_begin, uint32_t n_layers, uint32_t pages_per_tile,
                       uint64_t addr_or, int ctas, void* stream);

/* Affine launch form of a descriptor list: one query's consecutive chunks
 * (one page table, consecutive page-table columns, equally spaced chunk
 * bases, one layer stride, every descriptor full but the last). The unit
 * kernel then derives every address from the launch parameters, so the
 * page-table entry is the only load in front of the data — the layerwise
 * connector's one-layer launches take this form (same replaced reference
 * functions as tkv_gather_layers / tkv_scatter_layers). tkv_affine_form
 * returns 0 and fills *out when the HOST copy of the descriptors has the
 * form, TKV_NOT_FOUND otherwise. The affine launches need 16-byte-aligned
 * rows and bases and one plane (token_stride == bpt); any size. */
typedef struct tkv_affine_plan {
    uint32_t n_desc;
    uint32_t pages_per_desc;
    uint32_t last_tokens;
    uint32_t first_page;
    const int32_t* table_dev;
    uint32_t table_stride;
    uint32_t pad;
    uint64_t chunk0;
    uint64_t chunk_stride;
    uint64_t layer_stride;
} tkv_affine_plan;
int tkv_affine_form(const tkv_xfer_desc* descs, uint32_t n, uint32_t page_tokens, tkv_affine_plan* out);
int tkv_gather_layers_affine(const tkv_paged_layout* layout, const tkv_affine_plan* plan, uint32_t layer_begin,
                             uint32_t n_layers, int ctas, void* stream);
int tkv_scatter_layers_affine(const tkv_paged_layout* layout, const tkv_affine_plan* plan, uint32_t layer_begin,
                              uint32_t n_layers, int ctas, void* stream);

/* K3: one chained SHA-256 key sequence per chain (KeyChain::next,
 * src/tokens.cpp:22-42). out_dev gets 32 bytes per chunk at rows
 * out_first.. of each chain. tag_len <= 256. */
typedef struct tkv_chain_desc {
    uint64_t token_off;
    uint32_t n_tokens;
    uint32_t out_first;
    uint8_t parent[32];
} tkv_chain_desc;
int tkv_hash_chains(const uint32_t* tokens_dev, const tkv_chain_desc* chains_dev, uint32_t n_chains,
                    uint32_t chunk_size, const char* tag, uint32_t tag_len, uint8_t* out_dev,
                    void* stream);

/* K4: synth_token_kv (src/synth.cpp:7-20) into pages for positions
 * [pos_begin, pos_end) and layers [layer_begin, layer_end). */
int tkv_synth_pages(const tkv_paged_layout* layout, const uint32_t* tokens_dev,
                    const int32_t* table_dev, uint32_t table_stride, uint64_t seed,
                    uint32_t pos_begin, uint32_t pos_end, uint32_t layer_begin,
                    uint32_t layer_end, void* stream);
/* Adds the number of 8-byte words differing from synth to *mismatches_dev. */
int tkv_verify_pages(const tkv_paged_layout* layout, const uint32_t* tokens_dev,
                     const int32_t* table_dev, uint32_t table_stride, uint64_t seed,
                     uint32_t pos_begin, uint32_t pos_end, uint32_t layer_begin,
                     uint32_t layer_end, unsigned long long* mismatches_dev, void* stream);
/* Synthetic chunk payload [n_layers][n][bpt] (KVChunk layout, kv_chunk.hpp:12-36). */
int tkv_synth_chunk(const uint32_t* tokens_dev, uint64_t seed, uint32_t start, uint32_t n,
                    uint32_t n_layers, uint32_t bpt, uint8_t* out_dev, void* stream);

/* SM-driven copy of `bytes` from src to dst, both device-visible (HBM, mapped
 * or UVA pinned host memory, peer memory), on `stream`. For the engine's small
 * per-step uploads (prompt tokens): a kernel over PCIe never waits behind the
 * KV transfers queued on the copy engines. No reference equivalent (the
 * reference has no device). */
int tkv_sm_copy(const void* src, void* dst, uint64_t bytes, void* stream);
/* Copy-engine copy of `bytes` between any two device-visible addresses
 * (cudaMemcpyAsync, kind Default) on `stream`: the link probes (PCIe, NVLink
 * peer copy) the bench reports its rooflines against. */
int tkv_ce_copy(const void* src, void* dst, uint64_t bytes, void* stream);
/* Copy-engine copies of n pieces dst[i] <- src[i] (sizes[i] bytes) on
 * `stream`, grouped into pitched runs: pieces whose addresses both advance by
 * one constant step go as one 2D copy. `kind` is a cudaMemcpyKind value
 * (1 host->device, 2 device->host). The connector's host-tier path (a
 * layer's chunk slices in their slots). */
int tkv_ce_copy_pieces(void* const* dst, const void* const* src, const size_t* sizes, size_t n,
                       int kind, void* stream);
/* The grouping tkv_ce_copy_pieces applies (host only, no device call): fills
 * first[k], rows[k] for each run k (capacity n) and returns the run count.
 * Pitches above pitch_max never form a run. */
size_t tkv_plan_copy_runs(void* const* dst, const void* const* src, const size_t* sizes, size_t n,
                          size_t pitch_max, size_t* first, size_t* rows);

/* q8-scale codec (Q8ScaleCodec, src/codec.cpp:27-91), bit-exact, over a
 * batch of payloads. Encode: src = payload, dst = blob, bytes = payload
 * length; blob = u32 len | f32 scale | int8 lanes | odd tail byte
 * (tkv_q8_blob_bytes). Decode: src = blob, dst = payload, bytes = original
 * length. seg_base (n+1 entries) comes from tkv_codec_plan; scratch_dev
 * (the maxabs_dev argument) is tkv_q8_encode_scratch_bytes(n) bytes of
 * device scratch per call — per-item absmax and the single-pass encode's two
 * per-item counters — and must not be shared by encodes that may run
 * concurrently. */
typedef struct tkv_codec_item {
    const uint8_t* src_dev;
    uint8_t* dst_dev;
    uint64_t bytes;
} tkv_codec_item;
uint64_t tkv_q8_blob_bytes(uint64_t payload_bytes);
uint64_t tkv_q8_encode_scratch_bytes(uint32_t n);
int tkv_codec_plan(const tkv_codec_item* items, uint32_t n, uint32_t* seg_base_out);
int tkv_q8_encode(const tkv_codec_item* items_dev, const uint32_t* seg_base_dev, uint32_t n,
                  uint32_t total_segs, int* maxabs_dev, void* stream);
int tkv_q8_decode(const tkv_codec_item* items_dev, const uint32_t* seg_base_dev, uint32_t n,
                  uint32_t total_segs, void* stream);

/* ========================================================================== *
 * 2. Object level
 * ========================================================================== */

/* Chunk keys of one token sequence computed on the device (chunk_keys,
 * src/tokens.cpp:49-57). Writes n_chunks*32 bytes. */
int tkv_chunk_keys(const char* model_tag, size_t chunk_size, const uint32_t* tokens, size_t n,
                   uint8_t* digests_out, size_t* n_chunks);
/* One KeyChain link after reset(parent) (src/tokens.cpp:22-47). */
int tkv_keychain_next(const char* model_tag, size_t chunk_size, const uint8_t* parent,
                      const uint32_t* tokens, size_t n, uint8_t* digest_out);

/* ---- PagedKVStore (include/tierkv/paged_store.hpp:19-60) ----------------- */
typedef struct tkv_pages tkv_pages;
int tkv_pages_create(const tkv_model_spec* spec, uint32_t num_pages, int device, tkv_pages** out);
void tkv_pages_destroy(tkv_pages* p);
int tkv_pages_alloc(tkv_pages* p, uint64_t query, size_t n, uint32_t* ids_out);
int tkv_pages_bind_layer(tkv_pages* p, uint64_t query, uint32_t layer, const uint32_t* ids,
                         size_t n);
/* SimEngine::admit (src/sim_engine.cpp:83-95): allocate ceil(tokens/page)*L
 * pages and bind layer l to the l-th block run. */
int tkv_pages_admit(tkv_pages* p, uint64_t query, size_t tokens);
size_t tkv_pages_layer_pages(tkv_pages* p, uint64_t query, uint32_t layer, uint32_t* ids_out,
                             size_t cap);
size_t tkv_pages_release(tkv_pages* p, uint64_t query);
size_t tkv_pages_free_count(tkv_pages* p);
size_t tkv_pages_allocated_count(tkv_pages* p);
size_t tkv_pages_pool_pages(tkv_pages* p);
int tkv_pages_mark_populated(tkv_pages* p, uint32_t page, uint32_t layer);
int tkv_pages_populated(tkv_pages* p, uint32_t page);
/* Synchronous host-buffer gather/scatter of one layer (reference semantics
 * and checks; ordered after all previously enqueued device work). */
int tkv_pages_gather(tkv_pages* p, const uint32_t* ids, size_t n_ids, uint32_t layer,
                     size_t token_count, uint8_t* out, size_t out_bytes);
int tkv_pages_scatter(tkv_pages* p, const uint8_t* buf, size_t buf_bytes, const uint32_t* ids,
                      size_t n_ids, uint32_t layer, size_t token_count);
int tkv_pages_layout(tkv_pages* p, tkv_paged_layout* out);
int tkv_pages_device_table(tkv_pages* p, uint64_t query, void* stream, const int32_t** table_dev,
                           uint32_t* stride);
/* Tensor parallelism: this pool holds bytes [byte_offset, byte_offset + bpt)
 * of every full KV row (a head shard); the compute stand-in and its verifier
 * then produce / check exactly that slice of synth_token_kv's row. */
int tkv_pages_set_shard(tkv_pages* p, uint64_t byte_offset);
/* Engine compute stand-in (SimEngine::write_tokens, src/sim_engine.cpp:43-64):
 * K4 into the query's pages for positions [from, to), layers [l0, l1), and
 * marks them populated. tokens_dev holds the whole prompt. */
int tkv_pages_compute(tkv_pages* p, uint64_t query, const uint32_t* tokens_dev, uint32_t from,
                      uint32_t to, uint32_t layer_begin, uint32_t layer_end, void* stream);
/* Device byte oracle over [from, to) x [l0, l1): adds mismatching words. */
int tkv_pages_verify(tkv_pages* p, uint64_t query, const uint32_t* tokens_dev, uint32_t from,
                     uint32_t to, uint32_t layer_begin, uint32_t layer_end,
                     unsigned long long* mismatches_dev, void* stream);

/* ---- TieredStore RAM tier (include/tierkv/store.hpp:142-262) ------------- */
typedef struct tkv_store tkv_store;
int tkv_store_create(const tkv_model_spec* spec, size_t chunk_size, size_t ram_pool_bytes,
                     tkv_store** out);
void tkv_store_destroy(tkv_store* s);
int tkv_store_put(tkv_store* s, const uint8_t* digest, uint32_t token_count,
                  const uint8_t* payload, size_t payload_bytes, int pin);
int tkv_store_get(tkv_store* s, const uint8_t* digest, uint8_t* out, size_t cap, size_t* n);
int tkv_store_get_layer(tkv_store* s, const uint8_t* digest, uint32_t layer, uint8_t* out,
                        size_t cap, size_t* n);
int tkv_store_contains(tkv_store* s, const uint8_t* digest);
int tkv_store_pin(tkv_store* s, const uint8_t* digest, int on);
int tkv_store_clear(tkv_store* s, const uint8_t* digests, size_t n, size_t* removed,
                    size_t* refused);
/* Device byte oracle over one tier entry (test / bench verification, not a
 * reference API): the SMs read the chunk's pinned slot ([L][T][bpt]) over
 * PCIe and compare it with synth for tokens [start, start + T) of tokens_dev
 * (row slice at row_offset of the full row, TP shard), adding mismatching
 * 8-byte words to *mismatches_dev. Returns not_found for an absent chunk;
 * synchronizes `stream` before returning. */
int tkv_store_verify_synth(tkv_store* s, const uint8_t* digest, const uint32_t* tokens_dev, uint64_t seed,
                           uint32_t start, uint64_t row_offset, unsigned long long* mismatches_dev,
                           void* stream);
/* entries, ram_slots_total, ram_slots_used, ram_entries */
int tkv_store_stats(tkv_store* s, size_t out[4]);
/* LMCK records (chunk_file.hpp:12-56): export a present chunk / import a
 * record (checksum + geometry verified; corrupt_chunk / invalid_argument as
 * the reference). tkv_model_tag_hash = first 8 LE bytes of SHA-256(tag)
 * (hash.cpp:41-44), computed on the device. tkv_record_peek reads the
 * header: digest, {token_count, num_layers, bytes_per_token}, tag hash.
 * Export always sets *n to the record size; it writes the record only when
 * out != NULL and cap >= *n (a size query costs no copy or checksum). */
int tkv_model_tag_hash(const char* tag, uint64_t* out);
int tkv_store_export_record(tkv_store* s, const uint8_t* digest, uint64_t model_tag_hash,
                            uint8_t* out, size_t cap, size_t* n);
int tkv_store_import_record(tkv_store* s, const uint8_t* record, size_t n, int pin);
int tkv_record_peek(const uint8_t* record, size_t n, uint8_t* digest_out, uint32_t* geometry3,
                    uint64_t* model_tag_hash);

/* ---- Connector (include/tierkv/connector.hpp:74-152) --------------------- */
typedef struct tkv_connector tkv_connector;
typedef struct tkv_meta tkv_meta;
typedef struct tkv_connector_config {
    int layerwise;               /* TransferMode: 1 layerwise, 0 blocking */
    int pin_stores;
    size_t staging_budget_bytes; /* one layer of loads must fit, else blocking */
    uint32_t staging_depth;      /* device staging ring depth (layers) */
    int load_zero_copy;          /* 1: K2 reads pinned slots directly */
    int store_zero_copy;         /* 1: K1 writes pinned slots directly; 0: HBM ring + CE D2H */
    int store_ctas;              /* K1 grid for zero-copy stores (0 = default) */
    int load_ctas;               /* K2 grid (0 = 2 x SMs) */
    void* engine_stream;         /* stream the engine computes on */
    size_t memo_entries;         /* device prefix-digest memo links (0 = off) */
} tkv_connector_config;
void tkv_connector_config_default(tkv_connector_config* cfg);
int tkv_connector_create(tkv_store* s, tkv_pages* p, const tkv_connector_config* cfg,
                         tkv_connector** out);
/* Handles are reference-counted: a connector keeps its store and pages alive
   and a tkv_meta keeps its connector alive, so destroy calls may come in any
   order; the objects go when their last handle does. */
void tkv_connector_destroy(tkv_connector* c);
int tkv_connector_get_num_new_matched_tokens(tkv_connector* c, uint64_t query,
                                             const uint32_t* tokens, size_t n, size_t* matched);
int tkv_connector_lookup_batch(tkv_connector* c, size_t n_queries, const uint64_t* queries,
                               const uint32_t* const* prompts, const size_t* lens,
                               size_t* matched_out);
int tkv_connector_update_state_after_alloc(tkv_connector* c, uint64_t query, size_t blocks,
                                           size_t num_external_blocks);
int tkv_connector_build_meta(tkv_connector* c, size_t n_queries, const uint64_t* queries,
                             const uint32_t* const* prompts, const size_t* lens, tkv_meta** out);
int tkv_connector_start_load_kv(tkv_connector* c, tkv_meta* m);
int tkv_connector_wait_load_kv(tkv_connector* c, tkv_meta* m, uint32_t layer);
int tkv_connector_start_store_kv(tkv_connector* c, tkv_meta* m);
int tkv_connector_wait_store_kv(tkv_connector* c, tkv_meta* m, uint32_t layer);
/* Connector::prefetch / drain_prefetch (connector.hpp:96-99): promote
 * matched chunks from slower tiers; the pinned RAM tier is the only tier
 * here, so both return at once (kept for API parity). */
int tkv_connector_prefetch(tkv_connector* c, const uint32_t* tokens, size_t n);
int tkv_connector_drain_prefetch(tkv_connector* c);
int tkv_connector_begin_decode(tkv_connector* c, uint64_t query);
int tkv_connector_append_decode(tkv_connector* c, uint64_t query, uint32_t token);
/* One decode step of many queries: tokens[i] appended to queries[i];
 * statuses[i] = what tkv_connector_append_decode would return. */
int tkv_connector_append_decode_batch(tkv_connector* c, size_t n, const uint64_t* queries,
                                      const uint32_t* tokens, int* statuses);
int tkv_connector_finish_query(tkv_connector* c, uint64_t query, uint8_t* digests_out, size_t cap,
                               size_t* n);
size_t tkv_connector_staging_peak(tkv_connector* c);
/* Host-tier copy-engine traffic so far: out[0] = chunk-layer pieces copied,
 * out[1] = copies issued for them (pieces at a constant slot / ring pitch go
 * as one pitched copy). */
void tkv_connector_copy_runs(tkv_connector* c, uint64_t out[2]);
/* Prefix-digest memo counters: hits, misses (chunk links), capacity, resets,
 * re-hashed launches (a hit failed verification). */
int tkv_connector_memo_stats(tkv_connector* c, uint64_t out[5]);
/* Test hook: corrupt every memo slot's digest (verification must catch it). */
int tkv_connector_debug_poison_memo(tkv_connector* c);
uint64_t tkv_connector_hash_launches(tkv_connector* c);
/* Prompts whose stored prefix the host had to decide (the device presence
 * index decides the rest in the lookup launches): a memo hit that failed
 * verification, or a stored chunk the memo had no link for. */
uint64_t tkv_connector_lookups_host_decided(tkv_connector* c);
/* Lookup rows decided absent by the absence witness (no SHA-256 computed):
 * no present digest of the tier has that row's prefix. */
uint64_t tkv_connector_lookups_witnessed(tkv_connector* c);

void tkv_meta_destroy(tkv_meta* m);
int tkv_meta_layerwise(tkv_meta* m);
size_t tkv_meta_loaded_tokens(tkv_meta* m, uint64_t query);
size_t tkv_meta_num_plans(tkv_meta* m);
/* kind 0 = load plan, 1 = store plan; spans4 = (start, end, record_tokens,
 * chunk_index) per descriptor; digests 32 B each. */
int tkv_meta_plan(tkv_meta* m, size_t plan_index, int kind, uint64_t* spans4, uint8_t* digests,
                  size_t cap, size_t* n, uint64_t* matched);
int tkv_meta_store_results(tkv_meta* m, uint64_t query, int* codes, uint8_t* digests, size_t cap,
                           size_t* n);
/* Diagnostics: per layer {h2d done, load done, compute done, gathered, d2h
 * done} in ms since the batch's loads were enqueued (-1 = unused). Writes
 * 5*num_layers floats after the batch completed. */
int tkv_meta_timeline(tkv_meta* m, float* out, size_t cap, size_t* n);
/* Diagnostics: ms from the caller's completed timing event `cuda_event`
 * (a cudaEvent_t) to the batch's timeline origin (-1 if unavailable). */
int tkv_meta_origin_since(tkv_meta* m, void* cuda_event, float* ms);

/* ---- PD disaggregation over NVLink (run_pd, src/sim_engine.cpp:347-543;
 *      PdStaging, include/tierkv/pd_staging.hpp) --------------------------- */
typedef struct tkv_pd_staging tkv_pd_staging;
/* Where one pushed chunk landed on the decoder GPU ([L][T][bpt] payload). */
typedef struct tkv_pd_record {
    uint64_t addr;
    uint64_t bytes;
    uint32_t token_count;
    uint32_t first_token;
} tkv_pd_record;
int tkv_pd_staging_create(tkv_pd_staging** out);
void tkv_pd_staging_destroy(tkv_pd_staging* s);
int tkv_pd_register(tkv_pd_staging* s, uint64_t query);
/* Fills `ordinal` exactly once (duplicates ack); protocol_error on a push
 * beyond the final ordinal or a final marker below a filled one. */
int tkv_pd_push(tkv_pd_staging* s, uint64_t query, uint32_t ordinal, int last,
                const tkv_pd_record* rec);
/* Blocks until complete; records in ordinal order; forgets the query. */
int tkv_pd_await(tkv_pd_staging* s, uint64_t query, tkv_pd_record* out, size_t cap, size_t* n);
int tkv_pd_cancel(tkv_pd_staging* s, uint64_t query);
size_t tkv_pd_registered(tkv_pd_staging* s);
/* Prefiller: K1 of the query's first n_tokens (all chunks, all layers) from
 * `src` pages into landing_dev (chunk i at landing_dev + i*chunk_stride; may
 * be a peer GPU's memory). Returns when the bytes landed; fills the records
 * to push. */
int tkv_pd_send(tkv_pages* src, uint64_t query, size_t n_tokens, size_t chunk_size,
                uint64_t landing_dev, uint64_t chunk_stride, void* stream, tkv_pd_record* out,
                size_t cap, size_t* n);
/* Same contract through the copy engines: K1 gathers groups of chunks into
 * staging_dev (local HBM, chunk i at staging_dev + i*chunk_stride) while the
 * copy engine moves each finished group (about group_bytes; 0 = 1 GiB) to
 * landing_dev with one peer memcpy. Records point into landing_dev. */
/* Layer-streamed PD send (run_pd, src/sim_engine.cpp:389-424): one record
 * per unit of unit_tokens tokens — chunk_size (PdGranularity::chunk) or
 * page_tokens (PdGranularity::page) — at landing + i * unit_stride, laid out
 * [L][T_unit][bpt]. tkv_pd_sender_layer(l) gathers layer l of every unit into
 * the landing buffer, ordered after the work already queued on
 * engine_stream (the prefill's compute of layer l), on the sender's own
 * stream; finish waits for every layer (invalid_argument if one was not
 * sent) and returns the records to push to the decoder's PdStaging. The
 * landing memory must be ready before the first layer (the sender's stream
 * is ordered only after engine_stream). */
typedef struct tkv_pd_sender tkv_pd_sender;
int tkv_pd_sender_begin(tkv_pages* src, uint64_t query, size_t n_tokens, size_t unit_tokens, uint64_t landing,
                        uint64_t unit_stride, tkv_pd_sender** out);
int tkv_pd_sender_layer(tkv_pd_sender* s, uint32_t layer, void* engine_stream);
int tkv_pd_sender_finish(tkv_pd_sender* s, tkv_pd_record* out, size_t cap, size_t* n);
void tkv_pd_sender_destroy(tkv_pd_sender* s);
int tkv_pd_send_staged(tkv_pages* src, uint64_t query, size_t n_tokens, size_t chunk_size,
                       uint64_t landing_dev, uint64_t chunk_stride, uint64_t staging_dev,
                       uint64_t group_bytes, void* stream, tkv_pd_record* out, size_t cap, size_t* n);
/* Decoder: K2 of every landed record into the query's pages (one launch). */
int tkv_pd_land(tkv_pages* dst, uint64_t query, const tkv_pd_record* recs, size_t n, void* stream);
int tkv_enable_peer_access(int device, int peer);
/* CUDA IPC for cross-process landing buffers (one process per GPU). */
/* A handle names the whole allocation that contains dev_ptr; offset_out is
 * dev_ptr's offset in it (non-zero for sub-allocations of a caching
 * allocator). open maps the allocation and returns base + offset. */
int tkv_ipc_get_handle(void* dev_ptr, uint8_t* handle64, uint64_t* offset_out);
int tkv_ipc_open_handle(const uint8_t* handle64, uint64_t offset, void** dev_ptr_out);
int tkv_ipc_close(void* dev_ptr, uint64_t offset);

#ifdef __cplusplus
}
#endif

#endif /* TIERKV_B200_H */
