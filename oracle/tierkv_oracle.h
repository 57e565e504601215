/* TEST INFRASTRUCTURE ONLY — the CPU restatement ("oracle") of the reference
 * tierkv hot-path arithmetic. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker; the
 * product (paper_2510_09665_b200) never links or calls it.
 *
 * Parity pin: checked against the SURVEY.md Appendix A golden vectors and
 * against fixtures produced by the unmodified reference compiled from
 * /root/reference/proj/src (tests/golden/, tests/golden/make_golden.py).
 * Every function cites the reference file:line it restates.
 */
#ifndef TIERKV_ORACLE_H
#define TIERKV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FIPS 180-4 SHA-256 (reference: OpenSSL EVP via src/hash.cpp:9-29). */
void tkvo_sha256(const uint8_t* data, size_t n, uint8_t out[32]);

/* KeyChain::next, src/tokens.cpp:22-42:
 * SHA-256(u16le(taglen) | tag | parent[32] | u32le tokens[0..n)). */
void tkvo_keychain_next(const char* tag, size_t taglen, const uint8_t parent[32],
                        const uint32_t* tokens, size_t n, uint8_t out[32]);

/* chunk_keys, src/tokens.cpp:49-57 (with chunk_tokens, :7-15). Returns the
 * chunk count; writes count*32 digest bytes. */
size_t tkvo_chunk_keys(const uint32_t* tokens, size_t n, size_t chunk_size, const char* tag,
                       size_t taglen, uint8_t* out);

/* longest_prefix_match, src/tokens.cpp:59-69, KeyIndex = membership in an
 * unordered digest list (test_tokens.cpp:22-31). */
size_t tkvo_longest_prefix_match(const uint32_t* tokens, size_t n, size_t chunk_size,
                                 const char* tag, size_t taglen, const uint8_t* digests,
                                 size_t n_digests);

/* common.hpp:172-186 */
uint64_t tkvo_fnv1a64(const uint8_t* data, size_t n);
uint64_t tkvo_splitmix64(uint64_t x);
/* synth.hpp:27-30: fnv1a64(model_tag) */
uint64_t tkvo_model_seed(const char* tag, size_t taglen);
/* hash.cpp:41-44: first 8 LE bytes of SHA-256(tag) */
uint64_t tkvo_model_tag_hash(const char* tag, size_t taglen);

/* synth_token_kv / synth_layer_kv, src/synth.cpp:7-30 */
void tkvo_synth_token_kv(uint64_t seed, uint32_t token, uint32_t layer, uint64_t pos,
                         uint8_t* out, size_t bpt);
void tkvo_synth_layer_kv(uint64_t seed, const uint32_t* tokens, size_t n, uint32_t layer,
                         uint64_t first_pos, size_t bpt, uint8_t* out);
/* Layer-major chunk payload [L][n][bpt] for tokens [start, start+n) — the
 * KVChunk byte contract (kv_chunk.hpp:12-36) the RAM slot holds
 * (store.cpp:343-345). */
void tkvo_synth_chunk(uint64_t seed, const uint32_t* prompt, size_t start, size_t n,
                      uint32_t num_layers, size_t bpt, uint8_t* out);

/* PagedKVStore::gather_tokens_into / scatter_tokens data movement,
 * src/paged_store.cpp:123-140 and :147-175 (checks are done by callers). */
void tkvo_gather_tokens(const uint8_t* pool, size_t page_bytes, const uint32_t* pages,
                        size_t n_pages, size_t bpt, size_t token_count, uint8_t* out);
void tkvo_scatter_tokens(uint8_t* pool, size_t page_bytes, const uint32_t* pages, size_t n_pages,
                         size_t bpt, size_t token_count, const uint8_t* in);

/* Q8ScaleCodec, src/codec.cpp:27-94: blob = u32le len | f32le scale |
 * int8 lanes | raw odd tail. Returns bytes written (encode) / 0 on a
 * malformed blob (decode writes `len` payload bytes). */
size_t tkvo_q8_encode(const uint8_t* payload, size_t n, uint8_t* blob);
size_t tkvo_q8_decode(const uint8_t* blob, size_t n, uint8_t* payload);

#ifdef __cplusplus
}
#endif

#endif
