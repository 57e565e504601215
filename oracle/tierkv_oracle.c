/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference tierkv
 * hot-path arithmetic. See tierkv_oracle.h for the contract and the parity
 * pin. Plain C99, single-threaded, no dependencies. */
#include "tierkv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- SHA-256, FIPS 180-4 §6.2 (reference: OpenSSL via src/hash.cpp) ---- */

static const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
    0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
    0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
    0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
    0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
    0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
    0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
    0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};

#define ROTR(x, n) (((x) >> (n)) | ((x) << (32 - (n))))

typedef struct {
    uint32_t h[8];
    uint8_t buf[64];
    size_t fill;
    uint64_t total;
} sha_ctx;

static void sha_compress(uint32_t h[8], const uint8_t* blk) {
    uint32_t w[64];
    for (int t = 0; t < 16; ++t)
        w[t] = ((uint32_t)blk[4 * t] << 24) | ((uint32_t)blk[4 * t + 1] << 16) |
               ((uint32_t)blk[4 * t + 2] << 8) | (uint32_t)blk[4 * t + 3];
    for (int t = 16; t < 64; ++t) {
        uint32_t s0 = ROTR(w[t - 15], 7) ^ ROTR(w[t - 15], 18) ^ (w[t - 15] >> 3);
        uint32_t s1 = ROTR(w[t - 2], 17) ^ ROTR(w[t - 2], 19) ^ (w[t - 2] >> 10);
        w[t] = w[t - 16] + s0 + w[t - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int t = 0; t < 64; ++t) {
        uint32_t t1 = hh + (ROTR(e, 6) ^ ROTR(e, 11) ^ ROTR(e, 25)) + ((e & f) ^ (~e & g)) +
                      K256[t] + w[t];
        uint32_t t2 = (ROTR(a, 2) ^ ROTR(a, 13) ^ ROTR(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
        hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

static void sha_init(sha_ctx* c) {
    static const uint32_t iv[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    memcpy(c->h, iv, sizeof iv);
    c->fill = 0;
    c->total = 0;
}

static void sha_update(sha_ctx* c, const uint8_t* p, size_t n) {
    c->total += n;
    while (n) {
        size_t take = 64 - c->fill;
        if (take > n) take = n;
        memcpy(c->buf + c->fill, p, take);
        c->fill += take;
        p += take;
        n -= take;
        if (c->fill == 64) {
            sha_compress(c->h, c->buf);
            c->fill = 0;
        }
    }
}

static void sha_final(sha_ctx* c, uint8_t out[32]) {
    uint64_t bits = c->total * 8;
    uint8_t pad = 0x80;
    sha_update(c, &pad, 1);
    uint8_t zero = 0;
    while (c->fill != 56) sha_update(c, &zero, 1);
    uint8_t len[8];
    for (int i = 0; i < 8; ++i) len[i] = (uint8_t)(bits >> (56 - 8 * i));
    sha_update(c, len, 8);
    for (int i = 0; i < 8; ++i) {
        out[4 * i] = (uint8_t)(c->h[i] >> 24);
        out[4 * i + 1] = (uint8_t)(c->h[i] >> 16);
        out[4 * i + 2] = (uint8_t)(c->h[i] >> 8);
        out[4 * i + 3] = (uint8_t)c->h[i];
    }
}

void tkvo_sha256(const uint8_t* data, size_t n, uint8_t out[32]) {
    sha_ctx c;
    sha_init(&c);
    sha_update(&c, data, n);
    sha_final(&c, out);
}

/* ---- key chain (src/tokens.cpp:22-69) ---------------------------------- */

void tkvo_keychain_next(const char* tag, size_t taglen, const uint8_t parent[32],
                        const uint32_t* tokens, size_t n, uint8_t out[32]) {
    sha_ctx c;
    sha_init(&c);
    /* put_string16 (common.hpp:150-154): u16le length, then the bytes. */
    uint8_t hdr[2] = {(uint8_t)(taglen & 0xff), (uint8_t)(taglen >> 8)};
    sha_update(&c, hdr, 2);
    sha_update(&c, (const uint8_t*)tag, taglen);
    sha_update(&c, parent, 32);
    for (size_t i = 0; i < n; ++i) {
        uint8_t le[4] = {(uint8_t)tokens[i], (uint8_t)(tokens[i] >> 8), (uint8_t)(tokens[i] >> 16),
                         (uint8_t)(tokens[i] >> 24)};
        sha_update(&c, le, 4);
    }
    sha_final(&c, out);
}

size_t tkvo_chunk_keys(const uint32_t* tokens, size_t n, size_t chunk_size, const char* tag,
                       size_t taglen, uint8_t* out) {
    uint8_t parent[32] = {0};
    size_t count = 0;
    for (size_t start = 0; start < n; start += chunk_size) {
        size_t len = n - start < chunk_size ? n - start : chunk_size;
        tkvo_keychain_next(tag, taglen, parent, tokens + start, len, out + 32 * count);
        memcpy(parent, out + 32 * count, 32);
        ++count;
    }
    return count;
}

static int in_set(const uint8_t* d, const uint8_t* set, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (memcmp(d, set + 32 * i, 32) == 0) return 1;
    return 0;
}

size_t tkvo_longest_prefix_match(const uint32_t* tokens, size_t n, size_t chunk_size,
                                 const char* tag, size_t taglen, const uint8_t* digests,
                                 size_t n_digests) {
    uint8_t parent[32] = {0}, d[32];
    size_t matched = 0;
    for (size_t start = 0; start < n; start += chunk_size) {
        size_t len = n - start < chunk_size ? n - start : chunk_size;
        tkvo_keychain_next(tag, taglen, parent, tokens + start, len, d);
        if (!in_set(d, digests, n_digests)) break;
        matched = start + len;
        memcpy(parent, d, 32);
    }
    return matched;
}

/* ---- mixing / synthetic KV (common.hpp:172-186, src/synth.cpp:7-30) ---- */

uint64_t tkvo_fnv1a64(const uint8_t* data, size_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n; ++i) {
        h ^= data[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

uint64_t tkvo_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

uint64_t tkvo_model_seed(const char* tag, size_t taglen) {
    return tkvo_fnv1a64((const uint8_t*)tag, taglen);
}

uint64_t tkvo_model_tag_hash(const char* tag, size_t taglen) {
    uint8_t d[32];
    tkvo_sha256((const uint8_t*)tag, taglen, d);
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | d[i];
    return v;
}

void tkvo_synth_token_kv(uint64_t seed, uint32_t token, uint32_t layer, uint64_t pos,
                         uint8_t* out, size_t bpt) {
    uint64_t base = tkvo_splitmix64(seed ^ ((uint64_t)token << 32) ^ ((uint64_t)layer << 16) ^
                                    tkvo_splitmix64(pos));
    size_t i = 0;
    for (; i + 8 <= bpt; i += 8) {
        uint64_t w = tkvo_splitmix64(base + i);
        for (int b = 0; b < 8; ++b) out[i + b] = (uint8_t)(w >> (8 * b)); /* little-endian */
    }
    if (i < bpt) {
        uint64_t w = tkvo_splitmix64(base + i);
        for (size_t b = 0; i + b < bpt; ++b) out[i + b] = (uint8_t)(w >> (8 * b));
    }
}

void tkvo_synth_layer_kv(uint64_t seed, const uint32_t* tokens, size_t n, uint32_t layer,
                         uint64_t first_pos, size_t bpt, uint8_t* out) {
    for (size_t t = 0; t < n; ++t)
        tkvo_synth_token_kv(seed, tokens[t], layer, first_pos + t, out + t * bpt, bpt);
}

void tkvo_synth_chunk(uint64_t seed, const uint32_t* prompt, size_t start, size_t n,
                      uint32_t num_layers, size_t bpt, uint8_t* out) {
    for (uint32_t l = 0; l < num_layers; ++l)
        tkvo_synth_layer_kv(seed, prompt + start, n, l, start, bpt, out + (size_t)l * n * bpt);
}

/* ---- q8-scale codec (src/codec.cpp:27-94) ------------------------------ */

static int16_t q8_lane(const uint8_t* p, size_t i) {
    return (int16_t)(uint16_t)(p[2 * i] | ((uint16_t)p[2 * i + 1] << 8));
}

size_t tkvo_q8_encode(const uint8_t* payload, size_t n, uint8_t* blob) {
    size_t lanes = n / 2;
    int32_t max_abs = 0;
    for (size_t i = 0; i < lanes; ++i) {
        int32_t v = q8_lane(payload, i);
        if (v < 0) v = -v;
        if (v > max_abs) max_abs = v;
    }
    float scale = (float)((double)max_abs / 127.0);
    uint32_t len = (uint32_t)n, sb;
    memcpy(&sb, &scale, 4);
    for (int i = 0; i < 4; ++i) {
        blob[i] = (uint8_t)(len >> (8 * i));
        blob[4 + i] = (uint8_t)(sb >> (8 * i));
    }
    for (size_t i = 0; i < lanes; ++i) {
        double q = scale > 0 ? round((double)q8_lane(payload, i) / scale) : 0.0;
        if (q > 127.0) q = 127.0;
        if (q < -127.0) q = -127.0;
        blob[8 + i] = (uint8_t)(int8_t)q;
    }
    if (n & 1) blob[8 + lanes] = payload[n - 1];
    return 8 + lanes + (n & 1);
}

size_t tkvo_q8_decode(const uint8_t* blob, size_t n, uint8_t* payload) {
    if (n < 8) return 0;
    uint32_t len = 0, sb = 0;
    for (int i = 3; i >= 0; --i) {
        len = (len << 8) | blob[i];
        sb = (sb << 8) | blob[4 + i];
    }
    float scale;
    memcpy(&scale, &sb, 4);
    size_t lanes = len / 2;
    if (n != 8 + lanes + (len & 1)) return 0;
    for (size_t i = 0; i < lanes; ++i) {
        double v = round((double)(int8_t)blob[8 + i] * (double)scale);
        /* std::max(-32768.0, v) then std::min(32767.0, v) (codec.cpp:65): the
           comparisons are false for NaN, so a NaN product becomes -32768 */
        v = (-32768.0 < v) ? v : -32768.0;
        v = (v < 32767.0) ? v : 32767.0;
        uint16_t lane = (uint16_t)(int16_t)v;
        payload[2 * i] = (uint8_t)(lane & 0xff);
        payload[2 * i + 1] = (uint8_t)(lane >> 8);
    }
    if (len & 1) payload[len - 1] = blob[n - 1];
    return len;
}

/* ---- paged data movement (src/paged_store.cpp:123-175) ----------------- */

void tkvo_gather_tokens(const uint8_t* pool, size_t page_bytes, const uint32_t* pages,
                        size_t n_pages, size_t bpt, size_t token_count, uint8_t* out) {
    size_t off = 0, remaining = token_count * bpt;
    for (size_t i = 0; i < n_pages && remaining; ++i) {
        size_t take = remaining < page_bytes ? remaining : page_bytes;
        memcpy(out + off, pool + (size_t)pages[i] * page_bytes, take);
        off += take;
        remaining -= take;
    }
}

void tkvo_scatter_tokens(uint8_t* pool, size_t page_bytes, const uint32_t* pages, size_t n_pages,
                         size_t bpt, size_t token_count, const uint8_t* in) {
    size_t off = 0, remaining = token_count * bpt;
    for (size_t i = 0; i < n_pages && remaining; ++i) {
        size_t put = remaining < page_bytes ? remaining : page_bytes;
        memcpy(pool + (size_t)pages[i] * page_bytes, in + off, put);
        off += put;
        remaining -= put;
    }
}
