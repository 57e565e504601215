// K3 — chained SHA-256 chunk keys, bit-exact with KeyChain::next
// (src/tokens.cpp:22-42) over OpenSSL SHA-256 (src/hash.cpp:9-29).
//
// Message of chunk i of a chain (put_string16 / put_le, common.hpp:92-164):
//     u16le(|tag|) | tag | digest_{i-1} (32 B, zeros for i = 0) | u32le tokens
// With the 12-character tag of the configs that is 46 + 4*256 = 1070 bytes =
// 17 SHA-256 blocks per 256-token chunk.
//
// Parallelism. The chain is serial: block 0 of chunk i holds digest_{i-1},
// so chunks of one sequence cannot be compressed in parallel. One warp owns
// one chain (request) and walks its chunks; independent requests fill the
// GPU. Within a chunk the message words of the token-only blocks are packed
// straight from the u32 token array with one byte-permute per word
// (PRMT), so only the header block and the padding block take the generic
// byte path. What can be parallel is the memo: it is keyed by a fingerprint
// of the whole prefix, so every chunk of every chain is probed at once and
// only the rows after a chain's first miss go through SHA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.hpp"

namespace tkv {
namespace {

__constant__ uint32_t kK[64] = {
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

__device__ __forceinline__ uint32_t rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__device__ __forceinline__ void compress(uint32_t h[8], uint32_t w[16]) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        uint32_t wt;
        if (t < 16) {
            wt = w[t];
        } else {
            const uint32_t w15 = w[(t - 15) & 15], w2 = w[(t - 2) & 15];
            const uint32_t s0 = rotr(w15, 7) ^ rotr(w15, 18) ^ (w15 >> 3);
            const uint32_t s1 = rotr(w2, 17) ^ rotr(w2, 19) ^ (w2 >> 10);
            wt = w[t & 15] + s0 + w[(t - 7) & 15] + s1;
            w[t & 15] = wt;
        }
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t t1 = hh + S1 + ch + kK[t] + wt;
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        hh = g;
        g = f;
        f = e;
        e = d + t1;
        d = c;
        c = b;
        b = a;
        a = t1 + S0 + mj;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d;
    h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

struct ChunkMsg {
    const uint32_t* tok;  // this chunk's tokens
    uint32_t n;           // tokens in this chunk
    uint32_t hdr;         // 2 + tag_len + 32: first token byte offset
    uint32_t len;         // message bytes = hdr + 4n
    uint32_t nblocks;     // padded blocks
};

// Generic message byte (header, parent, token, padding or length byte).
__device__ __forceinline__ uint32_t msg_byte(const ChunkMsg& m, const HashParams& P,
                                             const uint32_t parent[8], uint32_t o) {
    const uint32_t tl = P.tag_len;
    if (o < 2) return (tl >> (8 * o)) & 0xff;
    if (o < 2 + tl) return P.tag[o - 2];
    if (o < m.hdr) {
        const uint32_t j = o - 2 - tl;
        return (parent[j >> 2] >> (24 - 8 * (j & 3))) & 0xff;
    }
    if (o < m.len) {
        const uint32_t k = o - m.hdr;
        return (__ldg(m.tok + (k >> 2)) >> (8 * (k & 3))) & 0xff;
    }
    if (o == m.len) return 0x80;
    const uint32_t end = 64 * m.nblocks;
    if (o >= end - 8) {
        const uint64_t bits = uint64_t(m.len) * 8;
        return uint32_t(bits >> (8 * (end - 1 - o))) & 0xff;
    }
    return 0;
}

__device__ __forceinline__ void load_block(const ChunkMsg& m, const HashParams& P,
                                           const uint32_t parent[8], uint32_t blk, uint32_t w[16]) {
    const uint32_t o0 = 64 * blk;
    if (o0 >= m.hdr && o0 + 64 <= m.len) {
        // Token-only block: word at offset o = BE of stream bytes k..k+3,
        // k = o - hdr, which straddle tokens k>>2 and (k>>2)+1 when k & 3 != 0.
        const uint32_t k0 = o0 - m.hdr;
        const uint32_t sh = k0 & 3;
        const uint32_t sel = (sh + 3) | ((sh + 2) << 4) | ((sh + 1) << 8) | (sh << 12);
        const uint32_t* t = m.tok + (k0 >> 2);
        if (sh == 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i] = __byte_perm(__ldg(t + i), 0, 0x0123);
        } else {
            uint32_t cur = __ldg(t);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint32_t nxt = __ldg(t + i + 1);
                w[i] = __byte_perm(cur, nxt, sel);
                cur = nxt;
            }
        }
        return;
    }
#pragma unroll 1
    for (int i = 0; i < 16; ++i) {
        const uint32_t o = o0 + 4 * i;
        w[i] = (msg_byte(m, P, parent, o) << 24) | (msg_byte(m, P, parent, o + 1) << 16) |
               (msg_byte(m, P, parent, o + 2) << 8) | msg_byte(m, P, parent, o + 3);
    }
}

__global__ void __launch_bounds__(128)
hash_chains_kernel(const uint32_t* __restrict__ tokens, const ChainDesc* __restrict__ chains,
                   uint32_t n_chains, const HashParams P, uint8_t* __restrict__ out) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_chains) return;
    const ChainDesc cd = chains[c];
    uint32_t parent[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        parent[i] = (uint32_t(cd.parent[4 * i]) << 24) | (uint32_t(cd.parent[4 * i + 1]) << 16) |
                    (uint32_t(cd.parent[4 * i + 2]) << 8) | uint32_t(cd.parent[4 * i + 3]);
    const uint32_t hdr = 2 + P.tag_len + 32;
    uint32_t row = cd.out_first;
    for (uint32_t start = 0; start < cd.n_tokens; start += P.chunk_size, ++row) {
        ChunkMsg m;
        m.tok = tokens + cd.token_off + start;
        m.n = min(P.chunk_size, cd.n_tokens - start);
        m.hdr = hdr;
        m.len = hdr + 4 * m.n;
        m.nblocks = (m.len + 9 + 63) / 64;
        uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                         0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
#pragma unroll 1
        for (uint32_t b = 0; b < m.nblocks; ++b) {
            uint32_t w[16];
            load_block(m, P, parent, b, w);
            compress(h, w);
        }
        uint32_t* o = reinterpret_cast<uint32_t*>(out + 32ull * row);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            parent[i] = h[i];
            o[i] = __byte_perm(h[i], 0, 0x0123);  // digest bytes are big-endian words
        }
    }
}

// ---- warp-cooperative chains (chunk_size <= kWarpChunkMax) ----------------
//
// The compression is inherently serial, so its latency is the floor; what the
// thread-per-chain kernel adds on top is memory latency: each block's 16
// token loads sit on the critical path between compressions. Here warps own
// a chain: lanes stage the chunk's tokens, build every message word in shared
// memory in parallel and expand the schedules one block per lane, and then
// all lanes of the compressing warp run the same rounds (SIMT: the cost of
// one) reading K+W by broadcast.
constexpr int kWarpChunkMax = 256;  // the reference chunk size; larger chunks use the kernel above
constexpr int kMaxWords = ((2 + kMaxTagBytes + 32 + 4 * kWarpChunkMax + 9 + 63) / 64) * 16;
constexpr int kMaxBlocks = kMaxWords / 16;

// Message schedule of one block (FIPS 180-4 §6.2.2 step 1) folded with the
// round constants: out[t] = K[t] + W[t]. Independent of the chaining state,
// so one lane per block expands them all before the serial rounds start.
__device__ __forceinline__ void expand_block(const uint32_t* in, uint32_t* out) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        w[i] = in[i];
        out[i] = w[i] + kK[i];
    }
#pragma unroll
    for (int t = 16; t < 64; ++t) {
        const uint32_t w15 = w[(t - 15) & 15], w2 = w[(t - 2) & 15];
        const uint32_t s0 = rotr(w15, 7) ^ rotr(w15, 18) ^ (w15 >> 3);
        const uint32_t s1 = rotr(w2, 17) ^ rotr(w2, 19) ^ (w2 >> 10);
        const uint32_t wt = w[t & 15] + s0 + w[(t - 7) & 15] + s1;
        w[t & 15] = wt;
        out[t] = wt + kK[t];
    }
}

// The 64 rounds with K+W precomputed: only the state recurrence is serial.
// The round is arranged around its shortest dependent path. With
//   Yd_t = h_t + (K+W)_t + d_t      (h_t = e_{t-3}, d_t = a_{t-3}: known
//                                    three rounds ahead, prepared off the chains)
// and T1_t = e_{t+1} - d_t,
//   e_{t+1} = Sigma1(e_t) + Ch(e_t, f_t, g_t) + Yd_t              one IADD3
//   a_{t+1} = Sigma0(a_t) + (e_{t+1} + (Maj(a_t, b_t, c_t) - d_t))
// so each chain is SHF -> LOP3 -> one add per round and a trails e by one
// add. The adds off the e chain run on the FMA pipe as IMADs (a multiplier
// ptxas cannot see is 1, so it cannot turn them back into ALU-pipe IADD3s):
// the ALU pipe keeps the 6 SHF + 4 LOP3 + 1 IADD3 of a round.
// Measured one chain on one warp (tools/microbench_sha.cu,
// profiles/r02_k3_round.jsonl): 27.7 cycles per round; round 1's
// h + KW + S1 + Ch then d + T1 order 30.3, the Y / Yd order 30.0.
__constant__ uint32_t kOneC = 1u, kMinusOneC = 0xffffffffu;

__device__ __forceinline__ uint32_t mad_c(uint32_t x, uint32_t m, uint32_t y) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(m), "r"(y));
    return r;
}

__device__ __forceinline__ void compress_kw(uint32_t h[8], const uint32_t* kw) {
    const uint32_t one = kOneC, mone = kMinusOneC;
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    uint32_t yd = mad_c(mad_c(hh, one, kw[0]), one, d);
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t mjd = mad_c(d, mone, mj);  // Maj - d
        const uint32_t e_new = S1 + ch + yd;
        const uint32_t a_new = mad_c(S0, one, mad_c(e_new, one, mjd));
        if (t + 1 < 64) yd = mad_c(mad_c(g, one, kw[t + 1]), one, c);  // next round: h = g, d = c
        hh = g;
        g = f;
        f = e;
        e = e_new;
        d = c;
        c = b;
        b = a;
        a = a_new;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d;
    h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// ---- prefix-digest memo helpers (warp-cooperative) --------------------------

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// Slot = 8 u64 (64 B): [0] tagword = (tag40 << 24) | entry, [2..5] digest
// words (16-byte aligned for vector loads). 0 = empty, kBusy = being
// published. The digest rides in the slot so a probe is one memory round
// trip; the full comparison against the entry (parent, n, every token,
// digest) runs afterwards, in parallel over all hit chunks
// (memo_verify_kernel).
constexpr unsigned long long kBusy = ~0ull;
constexpr uint32_t kNoEntry = 0xffffffffu;

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ bool memo_probe(const MemoView& M, uint64_t key, uint32_t* digest,
                                           uint32_t* entry) {
    const uint64_t tag = (key >> 24) | 1u;
    uint32_t slot = uint32_t(key) & M.slot_mask;
    for (uint32_t p = 0; p <= M.slot_mask; ++p, slot = (slot + 1) & M.slot_mask) {
        const unsigned long long* sp = M.slots + 8ull * slot;
        const unsigned long long sv = ld_acquire(sp);
        if (sv == 0) return false;
        if (sv == kBusy || (sv >> 24) != tag) continue;
        const uint4 d0 = __ldcg(reinterpret_cast<const uint4*>(sp + 2));
        const uint4 d1 = __ldcg(reinterpret_cast<const uint4*>(sp + 4));
        digest[0] = d0.x; digest[1] = d0.y; digest[2] = d0.z; digest[3] = d0.w;
        digest[4] = d1.x; digest[5] = d1.y; digest[6] = d1.z; digest[7] = d1.w;
        *entry = uint32_t(sv & 0xffffffu);
        return true;
    }
    return false;
}

// ---- link index (MemoView::links): digest -> prefix key ---------------------
// slot states of the link and presence tables
constexpr uint32_t kSlotEmpty = 0, kSlotPresent = 1, kSlotGone = 2, kSlotClaim = 3;

// One thread; h = the digest as SHA state words. A digest already indexed is
// left alone (same digest, same prefix, same key); a full table drops it.
__device__ void link_insert(uint32_t* links, uint32_t mask, const uint32_t h[8], uint64_t key) {
    uint32_t b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) b[i] = __byte_perm(h[i], 0, 0x0123);
    uint32_t i = b[0] & mask;
    for (uint32_t n = 0; n <= mask;) {
        uint32_t* sp = links + 16ull * i;
        const uint32_t st = atomicAdd(sp + 8, 0u);
        if (st == kSlotEmpty) {
            if (atomicCAS(sp + 8, kSlotEmpty, kSlotClaim) == kSlotEmpty) {
#pragma unroll
                for (int k = 0; k < 8; ++k) sp[k] = b[k];
                sp[9] = uint32_t(key);
                sp[10] = uint32_t(key >> 32);
                __threadfence();
                atomicExch(sp + 8, kSlotPresent);
                return;
            }
            continue;
        }
        if (st == kSlotClaim) continue;
        bool eq = true;
#pragma unroll
        for (int k = 0; k < 8; ++k) eq &= __ldcg(sp + k) == b[k];
        if (eq) return;
        i = (i + 1) & mask;
        ++n;
    }
}

// The prefix key of a digest (bytes as words), if a link recorded it.
__device__ bool link_find(const uint32_t* links, uint32_t mask, const uint32_t b[8], uint64_t* key) {
    uint32_t i = b[0] & mask;
    for (uint32_t n = 0; n <= mask;) {
        const uint32_t* sp = links + 16ull * i;
        const uint32_t st = atomicAdd(const_cast<uint32_t*>(sp + 8), 0u);
        if (st == kSlotEmpty) return false;
        if (st == kSlotClaim) continue;  // being published: wait for it
        bool eq = true;
#pragma unroll
        for (int k = 0; k < 8; ++k) eq &= __ldcg(sp + k) == b[k];
        if (eq) {
            *key = uint64_t(__ldcg(sp + 9)) | (uint64_t(__ldcg(sp + 10)) << 32);
            return true;
        }
        i = (i + 1) & mask;
        ++n;
    }
    return false;
}

// ---- absence witness W (PresenceView::witness): prefix key -> count ---------
__device__ __forceinline__ unsigned long long witness_key(uint64_t key) { return key ? key : 1ull; }

__device__ void witness_add(const PresenceView& P, uint64_t key, int delta) {
    const unsigned long long k = witness_key(key);
    uint32_t i = uint32_t(k ^ (k >> 32)) & P.mask;
    for (uint32_t n = 0; n <= P.mask; ++n, i = (i + 1) & P.mask) {
        unsigned long long* sp = P.witness + 2ull * i;
        const unsigned long long old = atomicCAS(sp, 0ull, k);
        if (old == 0ull || old == k) {
            atomicAdd(reinterpret_cast<unsigned int*>(sp + 1), unsigned(delta));
            return;
        }
    }
}

// May the tier hold a digest whose prefix key is `key`? (false = certainly not)
__device__ bool witness_may_hold(const PresenceView& P, uint64_t key) {
    if (P.witness == nullptr || __ldcg(P.unknown) != 0u) return true;
    const unsigned long long k = witness_key(key);
    uint32_t i = uint32_t(k ^ (k >> 32)) & P.mask;
    for (uint32_t n = 0; n <= P.mask; ++n, i = (i + 1) & P.mask) {
        const unsigned long long* sp = P.witness + 2ull * i;
        const unsigned long long v = __ldcg(sp);
        if (v == 0ull) return false;
        if (v == k) return __ldcg(reinterpret_cast<const unsigned int*>(sp + 1)) != 0u;
    }
    return true;
}

__device__ __forceinline__ void memo_insert(const MemoView& M, const uint32_t* s_parent, const uint32_t* s_tok,
                                            uint32_t n, uint64_t key, uint32_t lane, const uint32_t h[8]) {
    unsigned int e = 0;
    if (lane == 0) e = atomicAdd(M.counter, 1u);
    e = __shfl_sync(0xffffffffu, e, 0);
    if (e >= M.entry_cap) return;  // full: the memo stops growing until reset
    uint32_t* ent = M.entries + uint64_t(e) * M.entry_words;
    if (lane < 8) ent[lane] = s_parent[lane];
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) ent[8 + i] = h[i];
        ent[16] = n;
    }
    for (uint32_t idx = lane; idx < n; idx += 32) ent[17 + idx] = s_tok[idx];
    __threadfence();
    __syncwarp();
    if (lane == 0) {
        const unsigned long long packed = (((key >> 24) | 1u) << 24) | e;
        uint32_t slot = uint32_t(key) & M.slot_mask;
        for (uint32_t p = 0; p <= M.slot_mask; ++p, slot = (slot + 1) & M.slot_mask) {
            unsigned long long* sp = M.slots + 8ull * slot;
            if (atomicCAS(sp, 0ull, kBusy) != 0ull) continue;
            uint4* d = reinterpret_cast<uint4*>(sp + 2);
            d[0] = make_uint4(h[0], h[1], h[2], h[3]);
            d[1] = make_uint4(h[4], h[5], h[6], h[7]);
            __threadfence();
            atomicExch(sp, packed);  // publish: readers acquire the tag, then the digest
            break;
        }
        if (M.links != nullptr) link_insert(M.links, M.link_mask, h, key);
    }
}

// ---- presence index probe (PresenceView, kernels.hpp) ----------------------
constexpr uint32_t kDecided = 0x80000000u;

// Slot states of the presence index (PresenceView): kSlot* above.

// Is the digest whose words (digest bytes, little-endian) are b[8] in the
// table? Tombstones keep probe runs contiguous; a slot's digest and state
// are read together (one 64-byte line).
__device__ __forceinline__ bool presence_has_words(const PresenceView& P, const uint32_t b[8]) {
    uint32_t i = b[0] & P.mask;
    for (uint32_t n = 0; n <= P.mask; ++n, i = (i + 1) & P.mask) {
        const uint4* sp = reinterpret_cast<const uint4*>(P.slots + 16ull * i);
        const uint4 d0 = __ldcg(sp), d1 = __ldcg(sp + 1), st = __ldcg(sp + 2);
        if (st.x == kSlotEmpty) return false;
        if (d0.x == b[0] && d0.y == b[1] && d0.z == b[2] && d0.w == b[3] && d1.x == b[4] && d1.y == b[5] &&
            d1.z == b[6] && d1.w == b[7])
            return st.x == kSlotPresent;
    }
    return false;
}

// The same for a digest given as SHA chaining words h[8] (bytes = bswap).
__device__ __forceinline__ bool presence_has(const PresenceView& P, const uint32_t h[8]) {
    uint32_t b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) b[i] = __byte_perm(h[i], 0, 0x0123);
    return presence_has_words(P, b);
}

// The witness side of a digest turning present (slot sp, digest b): its
// prefix key goes into W, or the digest is counted unknown.
__device__ __forceinline__ void witness_count_add(const PresenceView& P, uint32_t* sp, const uint32_t b[8]) {
    if (P.witness == nullptr) return;
    uint64_t key = 0;
    if (P.links != nullptr && link_find(P.links, P.link_mask, b, &key)) {
        sp[9] = uint32_t(key);
        sp[10] = uint32_t(key >> 32);
        sp[11] = 1;
        witness_add(P, key, 1);
    } else {
        sp[11] = 2;
        atomicAdd(P.unknown, 1u);
    }
}

// ... and of it turning absent: exactly what its add counted.
__device__ __forceinline__ void witness_count_remove(const PresenceView& P, const uint32_t* sp) {
    if (P.witness == nullptr) return;
    const uint32_t mode = __ldcg(sp + 11);
    if (mode == 1) witness_add(P, uint64_t(__ldcg(sp + 9)) | (uint64_t(__ldcg(sp + 10)) << 32), -1);
    else if (mode == 2) atomicSub(P.unknown, 1u);
}

// Applies one pending change (one thread per distinct digest): find the
// digest's slot in its probe run and set its state, or claim the run's first
// empty slot (CAS; a concurrent claimer of the same slot publishes its own
// digest, which we then compare and step past). Removing an absent digest is
// a no-op; slots are never reused within a table generation (the host
// rebuilds the table before the tombstones fill it). Only real transitions
// (absent -> present, present -> absent) touch the witness.
__device__ void presence_apply(const PresenceView& P, const uint32_t* u) {
    uint32_t b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) b[k] = u[k];
    const bool present = u[8] != 0;
    uint32_t i = b[0] & P.mask;
    for (uint32_t n = 0; n <= P.mask;) {
        uint32_t* sp = P.slots + 16ull * i;
        uint32_t st = atomicAdd(sp + 8, 0u);
        if (st == kSlotEmpty) {
            if (!present) return;
            if (atomicCAS(sp + 8, kSlotEmpty, kSlotClaim) == kSlotEmpty) {
#pragma unroll
                for (int k = 0; k < 8; ++k) sp[k] = b[k];
                witness_count_add(P, sp, b);
                __threadfence();
                atomicExch(sp + 8, kSlotPresent);
                return;
            }
            continue;  // lost the claim: re-read this slot
        }
        if (st == kSlotClaim) continue;  // another digest is being published here
        __threadfence();
        bool eq = true;
#pragma unroll
        for (int k = 0; k < 8; ++k) eq &= __ldcg(sp + k) == b[k];
        if (eq) {
            const uint32_t old = atomicExch(sp + 8, present ? kSlotPresent : kSlotGone);
            if (present && old != kSlotPresent) witness_count_add(P, sp, b);
            if (!present && old == kSlotPresent) witness_count_remove(P, sp);
            return;
        }
        i = (i + 1) & P.mask;
        ++n;
    }
}

// ---- producer / consumer variant: two warps per chain ----------------------
//
// The serial compression is ~83 % of a chunk (ncu source samples); the rest —
// staging tokens, building message words, expanding the message schedules —
// does not depend on the chaining state except for the block(s) holding the
// parent digest. So a second warp prepares chunk i+1 (tokens, words, K+W of
// every parent-free block) in a double buffer while the first compresses
// chunk i; the consumer only builds and expands the parent block(s) itself.
constexpr int kPairsPerCta = 2;

struct PairSmem {
    uint32_t tok[2][kWarpChunkMax + 4];
    uint32_t w[2][kMaxWords];
    uint32_t kw[2][kMaxBlocks * 64];
    uint32_t parent[8];
};

__device__ __forceinline__ void named_barrier(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Message byte o of a chunk (header, parent, token, padding or length byte).
__device__ __forceinline__ uint32_t pair_msg_byte(const uint32_t* tok, const uint32_t* parent, const HashParams& P,
                                                  uint32_t hdr, uint32_t len, uint32_t end, uint32_t o) {
    const uint32_t tl = P.tag_len;
    if (o < 2) return (tl >> (8 * o)) & 0xff;
    if (o < 2 + tl) return P.tag[o - 2];
    if (o < hdr) {
        const uint32_t j = o - 2 - tl;
        return (parent[j >> 2] >> (24 - 8 * (j & 3))) & 0xff;
    }
    if (o < len) {
        const uint32_t k = o - hdr;
        return (tok[k >> 2] >> (8 * (k & 3))) & 0xff;
    }
    if (o == len) return 0x80;
    if (o >= end - 8) return uint32_t((uint64_t(len) * 8) >> (8 * (end - 1 - o))) & 0xff;
    return 0;
}

// Word j (4 message bytes, big-endian) of a chunk; token-only words by PRMT.
__device__ __forceinline__ uint32_t pair_msg_word(const uint32_t* tok, const uint32_t* parent, const HashParams& P,
                                                  uint32_t hdr, uint32_t len, uint32_t end, uint32_t j) {
    const uint32_t o = 4 * j;
    if (o >= hdr && o + 4 <= len) {
        const uint32_t k = o - hdr;
        const uint32_t kk = k & 3;
        const uint32_t sl = (kk + 3) | ((kk + 2) << 4) | ((kk + 1) << 8) | (kk << 12);
        return __byte_perm(tok[k >> 2], kk ? tok[(k >> 2) + 1] : 0u, sl);
    }
    return (pair_msg_byte(tok, parent, P, hdr, len, end, o) << 24) |
           (pair_msg_byte(tok, parent, P, hdr, len, end, o + 1) << 16) |
           (pair_msg_byte(tok, parent, P, hdr, len, end, o + 2) << 8) |
           pair_msg_byte(tok, parent, P, hdr, len, end, o + 3);
}

__global__ void __launch_bounds__(64 * kPairsPerCta)
hash_chains_pair_kernel(const uint32_t* __restrict__ tokens, const ChainDesc* __restrict__ chains,
                        uint32_t n_chains, const HashParams P, uint8_t* __restrict__ out, const MemoView M) {
    __shared__ PairSmem smem[kPairsPerCta];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t pair = threadIdx.x >> 6;
    const bool producer = (threadIdx.x >> 5) & 1;
    const uint32_t c = blockIdx.x * kPairsPerCta + pair;
    if (c >= n_chains) return;  // both warps of the pair
    PairSmem& s = smem[pair];
    const ChainDesc cd = chains[c];
    const uint32_t cs = P.chunk_size;
    const uint32_t k0 = M.first_miss != nullptr ? M.first_miss[c] : 0u;
    const uint32_t start0 = k0 * cs;
    if (start0 >= cd.n_tokens) return;  // both warps
    uint32_t nchunks = (cd.n_tokens - start0 + cs - 1) / cs;
    if (M.max_rows) nchunks = min(nchunks, M.max_rows);
    const uint32_t hdr = 2 + P.tag_len + 32;
    const uint32_t pb0 = (2 + P.tag_len) / 64, pb1 = (hdr - 1) / 64;  // blocks holding the parent
    const uint32_t bar_id = 1 + pair;
    const uint32_t* base = tokens + cd.token_off;

    auto produce = [&](uint32_t j) {
        const uint32_t b = j & 1;
        const uint32_t start = start0 + j * cs;
        const uint32_t n = min(cs, cd.n_tokens - start);
        for (uint32_t idx = lane; idx < n; idx += 32) s.tok[b][idx] = __ldg(base + start + idx);
        if (lane == 0) s.tok[b][n] = 0;
        __syncwarp();
        const uint32_t len = hdr + 4 * n;
        const uint32_t nblocks = (len + 9 + 63) / 64;
        const uint32_t end = 64 * nblocks;
        for (uint32_t jw = lane; jw < 16 * nblocks; jw += 32) {
            const uint32_t blk = jw >> 4;
            if (blk >= pb0 && blk <= pb1) continue;  // parent block(s): the consumer's
            s.w[b][jw] = pair_msg_word(s.tok[b], nullptr, P, hdr, len, end, jw);
        }
        __syncwarp();
        for (uint32_t blk = lane; blk < nblocks; blk += 32)
            if (blk < pb0 || blk > pb1) expand_block(s.w[b] + 16 * blk, s.kw[b] + 64 * blk);
        __syncwarp();
    };

    if (producer) {
        produce(0);
    } else if (lane < 8) {
        s.parent[lane] =
            k0 ? __byte_perm(reinterpret_cast<const uint32_t*>(out + 32ull * (cd.out_first + k0 - 1))[lane], 0, 0x0123)
               : (uint32_t(cd.parent[4 * lane]) << 24) | (uint32_t(cd.parent[4 * lane + 1]) << 16) |
                     (uint32_t(cd.parent[4 * lane + 2]) << 8) | uint32_t(cd.parent[4 * lane + 3]);
    }
    unsigned long long misses = 0;
    for (uint32_t j = 0; j < nchunks; ++j) {
        named_barrier(bar_id, 64);  // chunk j prepared; the other buffer is free
        if (producer) {
            if (j + 1 < nchunks) produce(j + 1);
            continue;
        }
        const uint32_t b = j & 1;
        const uint32_t start = start0 + j * cs;
        const uint32_t n = min(cs, cd.n_tokens - start);
        const uint32_t len = hdr + 4 * n;
        const uint32_t nblocks = (len + 9 + 63) / 64;
        const uint32_t end = 64 * nblocks;
        const uint32_t row = cd.out_first + k0 + j;
        const uint64_t key = M.slots != nullptr ? M.keys[row] : 0;
        if (M.hit_entry != nullptr && lane == 0) M.hit_entry[row] = kNoEntry;
        ++misses;
        // parent block(s): words, then their schedules
        for (uint32_t jw = 16 * pb0 + lane; jw < 16 * (pb1 + 1); jw += 32)
            s.w[b][jw] = pair_msg_word(s.tok[b], s.parent, P, hdr, len, end, jw);
        __syncwarp();
        if (lane <= pb1 - pb0) expand_block(s.w[b] + 16 * (pb0 + lane), s.kw[b] + 64 * (pb0 + lane));
        __syncwarp();
        uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                         0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
#pragma unroll 1
        for (uint32_t blk = 0; blk < nblocks; ++blk) compress_kw(h, s.kw[b] + 64 * blk);
        __syncwarp();
        if (M.slots != nullptr) memo_insert(M, s.parent, s.tok[b], n, key, lane, h);  // needs the old parent
        __syncwarp();
        if (lane == 0) {
            uint32_t* o = reinterpret_cast<uint32_t*>(out + 32ull * row);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                s.parent[i] = h[i];
                o[i] = __byte_perm(h[i], 0, 0x0123);
            }
            // lookup mode: the row after the present memo hits was hashed;
            // its presence decides the prefix unless it is present too
            if (M.lookup.present_out != nullptr && M.presence.slots != nullptr && j == 0) {
                const uint32_t rows = (cd.n_tokens + cs - 1) / cs;
                const uint32_t k = k0 + 1;
                M.lookup.present_out[c] =
                    presence_has(M.presence, h) ? (k | (k == rows ? kDecided : 0u)) : ((k - 1) | kDecided);
            }
        }
        __syncwarp();
    }
    if (!producer && M.stats != nullptr && lane == 0 && misses) atomicAdd(M.stats + 1, misses);
}

// Largest chain index c with chains[c].out_first <= row.
__device__ __forceinline__ uint32_t chain_of_row(const ChainDesc* __restrict__ chains, uint32_t n_chains,
                                                 uint32_t row) {
    uint32_t lo = 0, hi = n_chains;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (chains[mid].out_first <= row) lo = mid; else hi = mid;
    }
    return lo;
}

// Memo pass 1, one warp per row of every chain: copies the row's tokens from
// the mapped host buffer into HBM (the copy the plain path does with
// stage_words_kernel) and writes the row's chunk fingerprint to keys[row].
// With chains_dst set, `chains` is the mapped host copy of at most
// kStageChains descriptors: every block reads them once into shared memory
// and block 0 also stages them into chains_dst for the later passes (one
// copy launch fewer per lookup).
constexpr uint32_t kStageChains = 128;

__global__ void __launch_bounds__(128)
memo_fingerprint_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                        const ChainDesc* __restrict__ chains, uint32_t n_chains, uint32_t total_rows,
                        const HashParams P, const MemoView M, ChainDesc* __restrict__ chains_dst,
                        const unsigned long long* __restrict__ chain_src) {
    __shared__ ChainDesc s_chains[kStageChains];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (chains_dst != nullptr) {
        const uint32_t words = n_chains * uint32_t(sizeof(ChainDesc) / 4);
        const uint32_t* cs = reinterpret_cast<const uint32_t*>(chains);
        uint32_t* sm = reinterpret_cast<uint32_t*>(s_chains);
        uint32_t* gd = reinterpret_cast<uint32_t*>(chains_dst);
        for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) {
            const uint32_t w = cs[i];
            sm[i] = w;
            if (blockIdx.x == 0) gd[i] = w;
        }
        __syncthreads();
        chains = s_chains;
    }
    // pending presence changes, applied before the probe kernel (next launch)
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < M.presence.n_updates; u += gridDim.x * blockDim.x)
        presence_apply(M.presence, M.presence.updates + 9ull * u);
    if (row >= total_rows) return;
    const uint32_t ci = chain_of_row(chains, n_chains, row);
    const ChainDesc& cd = chains[ci];
    const uint32_t k = row - cd.out_first;
    const uint32_t start = k * P.chunk_size;
    const uint32_t n = min(P.chunk_size, cd.n_tokens - start);
    const uint64_t off = cd.token_off + start;
    const uint32_t* s = chain_src != nullptr ? reinterpret_cast<const uint32_t*>(chain_src[ci]) + start : src + off;
    uint64_t h = 0;
    if (n == 256 && ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(dst + off)) & 15) == 0) {
        // a full row, 16-byte aligned: two 16-byte loads per lane (512-byte
        // requests per warp over PCIe instead of 128-byte ones)
        const uint4 v0 = reinterpret_cast<const uint4*>(s)[lane];
        const uint4 v1 = reinterpret_cast<const uint4*>(s)[32 + lane];
        reinterpret_cast<uint4*>(dst + off)[lane] = v0;
        reinterpret_cast<uint4*>(dst + off)[32 + lane] = v1;
        const uint32_t i0 = 4 * lane, i1 = 128 + 4 * lane;
        h = mix64((uint64_t(v0.x) << 32) | i0) ^ mix64((uint64_t(v0.y) << 32) | (i0 + 1)) ^
            mix64((uint64_t(v0.z) << 32) | (i0 + 2)) ^ mix64((uint64_t(v0.w) << 32) | (i0 + 3)) ^
            mix64((uint64_t(v1.x) << 32) | i1) ^ mix64((uint64_t(v1.y) << 32) | (i1 + 1)) ^
            mix64((uint64_t(v1.z) << 32) | (i1 + 2)) ^ mix64((uint64_t(v1.w) << 32) | (i1 + 3));
    } else if (n <= 256) {
        // all of a lane's tokens requested before any is used: the source is
        // mapped host memory, one PCIe round trip instead of eight
        uint32_t tv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t idx = lane + 32u * j;
            tv[j] = idx < n ? s[idx] : 0u;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t idx = lane + 32u * j;
            if (idx < n) {
                dst[off + idx] = tv[j];
                h ^= mix64((uint64_t(tv[j]) << 32) | idx);
            }
        }
    } else {
        for (uint32_t idx = lane; idx < n; idx += 32) {
            const uint32_t t = s[idx];
            dst[off + idx] = t;
            h ^= mix64((uint64_t(t) << 32) | idx);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, o);
    if (lane == 0)
        M.keys[row] = mix64(h ^ (uint64_t(n) * 0xc2b2ae3d27d4eb4full) ^ (uint64_t(k) * 0x9e3779b97f4a7c15ull));
}

// Memo pass 2, one CTA per chain: an inclusive scan of the row fingerprints
// over the chain (wrapping add, so key_k covers the parent and every token up
// to the end of chunk k), then one independent probe per row. Hits publish their digest to `out` and
// their entry to hit_entry (checked later by memo_verify_kernel); the first
// miss of the chain goes to first_miss, where the SHA chain resumes. Every
// row's key is kept for the insertions of the rows that miss.
constexpr int kProbeThreads = 1024;  // a 256K-token chain's rows in one tile

__global__ void __launch_bounds__(kProbeThreads)
memo_probe_kernel(const ChainDesc* __restrict__ chains, const HashParams P, uint8_t* __restrict__ out, const MemoView M) {
    __shared__ unsigned long long warp_sum[kProbeThreads / 32];
    __shared__ uint32_t first;   // first row the memo missed
    __shared__ uint32_t absent;  // first memo hit that is not in the tier (with a presence index)
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const ChainDesc cd = chains[blockIdx.x];
    const uint32_t cs = P.chunk_size;
    const uint32_t rows = (cd.n_tokens + cs - 1) / cs;
    unsigned long long* keys = M.keys + cd.out_first;
    if (threadIdx.x == 0) first = absent = rows;
    // lookup mode (hash_prefix with a presence index): presence decides too
    const bool lookup = M.lookup.present_out != nullptr && M.presence.slots != nullptr;
    // the chain's parent digest (KeyChain::reset) seeds every key of the chain
    uint64_t pfp = 0x8f1bbcdcca62c1d6ull;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint64_t w = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) w |= uint64_t(cd.parent[8 * i + b]) << (8 * b);
        pfp = mix64(pfp ^ w);
    }
    __syncthreads();
    // 2. scan + probe, one thread per row
    uint64_t carry = 0;
    for (uint32_t base = 0; base < rows; base += kProbeThreads) {
        const uint32_t k = base + threadIdx.x;
        uint64_t v = k < rows ? keys[k] : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint64_t t = __shfl_up_sync(0xffffffffu, v, off);
            if (lane >= uint32_t(off)) v += t;
        }
        if (lane == 31) warp_sum[wid] = v;
        __syncthreads();
        uint64_t before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kProbeThreads / 32; ++w) {
            const uint64_t ws = warp_sum[w];
            before += uint32_t(w) < wid ? ws : 0;
            total += ws;
        }
        v += before + carry;
        carry += total;
        const bool skip = min(first, absent) < base;  // an earlier tile already ended the prefix
        if (k < rows) {
            const uint64_t key = mix64(v ^ pfp);
            keys[k] = key;
            uint32_t d[8], ent = kNoEntry;
            if (!skip && memo_probe(M, key, d, &ent)) {
                uint32_t* o = reinterpret_cast<uint32_t*>(out + 32ull * (cd.out_first + k));
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] = __byte_perm(d[i], 0, 0x0123);
                if (lookup && !presence_has(M.presence, d)) atomicMin(&absent, k);
            } else {
                ent = kNoEntry;
                atomicMin(&first, k);
            }
            M.hit_entry[cd.out_first + k] = ent;
        }
        __syncthreads();  // warp_sum reuse; `first` settled for the next tile
    }
    if (threadIdx.x == 0) {
        if (lookup) {
            // the stored prefix, decided on the device: a memo hit that is not
            // in the tier ends it (no SHA needed); otherwise the first row the
            // memo missed is hashed (max_rows = 1) and its presence decides
            if (absent < first) {
                M.first_miss[blockIdx.x] = rows;  // nothing to hash
                M.lookup.present_out[blockIdx.x] = absent | kDecided;
                M.lookup.known_out[blockIdx.x] = absent + 1;
            } else if (first < rows && !witness_may_hold(M.presence, keys[first])) {
                // no present digest has this row's prefix: absent, no SHA
                if (M.stats != nullptr) atomicAdd(M.stats + 2, 1ull);
                M.first_miss[blockIdx.x] = rows;
                M.lookup.present_out[blockIdx.x] = first | kDecided;
                M.lookup.known_out[blockIdx.x] = first;
            } else {
                M.first_miss[blockIdx.x] = first;
                M.lookup.present_out[blockIdx.x] = first | (first >= rows ? kDecided : 0u);
                M.lookup.known_out[blockIdx.x] = min(rows, first + 1);
            }
        } else {
            M.first_miss[blockIdx.x] = first;
        }
        if (M.stats != nullptr && first) atomicAdd(M.stats, (unsigned long long)first);
    }
}

// One warp per digest row: a memo hit is checked against its entry (parent,
// token count, every token, digest); every row's digest is then published to
// the caller's buffer. A failed check records the first bad row of its chain
// (the host re-hashes that chain from there without the memo).
__global__ void __launch_bounds__(128)
memo_verify_kernel(const uint32_t* __restrict__ tokens, const ChainDesc* __restrict__ chains,
                   uint32_t n_chains, uint32_t total_rows, const HashParams P,
                   const uint8_t* __restrict__ dev_out, const MemoView M, uint8_t* __restrict__ out,
                   unsigned int* __restrict__ first_bad) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (M.first_miss_out != nullptr)  // publish the probe's first misses (saves a copy launch)
        for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n_chains; c += gridDim.x * blockDim.x)
            M.first_miss_out[c] = M.first_miss[c];
    if (row >= total_rows) return;
    const uint32_t dw = lane < 8 ? reinterpret_cast<const uint32_t*>(dev_out + 32ull * row)[lane] : 0u;
    if (lane < 8) reinterpret_cast<uint32_t*>(out + 32ull * row)[lane] = dw;
    if (M.hit_entry == nullptr) return;
    const uint32_t e = M.hit_entry[row];
    if (e == kNoEntry) return;
    const uint32_t lo = chain_of_row(chains, n_chains, row);
    const ChainDesc& cd = chains[lo];
    const uint32_t k = row - cd.out_first;
    const uint32_t start = k * P.chunk_size;
    const uint32_t n = min(P.chunk_size, cd.n_tokens - start);
    const uint32_t* ent = M.entries + uint64_t(e) * M.entry_words;
    const uint32_t* tok = tokens + cd.token_off + start;
    uint32_t bad = 0;
    if (lane < 8) {
        // parent of this row: previous row's digest, or the chain's parent
        const uint32_t parent = k ? __byte_perm(reinterpret_cast<const uint32_t*>(dev_out + 32ull * (row - 1))[lane], 0, 0x0123)
                                  : ((uint32_t(cd.parent[4 * lane]) << 24) | (uint32_t(cd.parent[4 * lane + 1]) << 16) |
                                     (uint32_t(cd.parent[4 * lane + 2]) << 8) | uint32_t(cd.parent[4 * lane + 3]));
        bad |= ent[lane] ^ parent;
        bad |= ent[8 + lane] ^ __byte_perm(dw, 0, 0x0123);
    }
    if (lane == 0) bad |= ent[16] ^ n;
    for (uint32_t idx = lane; idx < n; idx += 32) bad |= ent[17 + idx] ^ tok[idx];
    if (__any_sync(0xffffffffu, bad != 0) && lane == 0) atomicMin(first_bad + lo, k);
}

// ---- cold-lookup fast path: the first row of every chain, in one launch ----
// (FirstRowInline, kernels.hpp: a single chain's row-0 tokens as parameters)
//
// A lookup's stored prefix is empty when its first chunk is absent — the
// usual case for a new document. The full lookup stages the whole prompt and
// probes every row (four launches, ~0.1 ms for 128K tokens); this kernel
// decides row 0 alone from its 256 tokens: memo probe of the row's prefix
// key (verified against the entry), else the chunk's SHA-256 by one warp
// (inserting the link), then the presence index. Per chain it publishes the
// digest and a flag (bit 0: done, bit 1: present) to mapped memory with a
// system-scope release, so the host can poll instead of synchronizing and
// return at once when every chain's first chunk is absent.
constexpr int kFirstRowWarps = 2;
constexpr int kFirstRowMaxThreads = 256;  // chain warps + presence-apply warps

struct FirstRowSmem {
    uint32_t tok[kWarpChunkMax + 4];
    uint32_t w[kMaxWords];
    uint32_t kw[kMaxBlocks * 64];
    uint32_t parent[8];
};

__device__ __forceinline__ uint64_t parent_fingerprint(const uint8_t parent[32]) {
    uint64_t pfp = 0x8f1bbcdcca62c1d6ull;  // as memo_probe_kernel
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint64_t w = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) w |= uint64_t(parent[8 * i + b]) << (8 * b);
        pfp = mix64(pfp ^ w);
    }
    return pfp;
}

__global__ void __launch_bounds__(kFirstRowMaxThreads)
first_row_kernel(const uint32_t* __restrict__ tokens, const ChainDesc* __restrict__ chains, uint32_t n_chains,
                 const HashParams P, const MemoView M, uint32_t* __restrict__ digests_out,
                 uint32_t* __restrict__ flags_out, unsigned long long* __restrict__ trace, const FirstRowInline one) {
    __shared__ FirstRowSmem smem[kFirstRowWarps];
    __shared__ uint32_t applied_warps;
    unsigned long long t_start = 0, t_staged = 0, t_hashed = 0;
    if (trace != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // Pending presence changes (only in a one-CTA launch: the host launches
    // presence_apply_kernel first otherwise). Warps past the chain warps
    // apply them while the chain warps stage and hash; a chain warp waits for
    // them (shared counter) only before its presence test.
    const uint32_t apply_warps = blockDim.x / 32 - kFirstRowWarps;
    if (M.presence.n_updates != 0 && apply_warps == 0 && gridDim.x == 1) {
        for (uint32_t u = threadIdx.x; u < M.presence.n_updates; u += blockDim.x)
            presence_apply(M.presence, M.presence.updates + 9ull * u);
        __threadfence_block();
        __syncthreads();
    }
    if (apply_warps != 0) {
        if (threadIdx.x == 0) applied_warps = 0;
        __syncthreads();
        if (wid >= uint32_t(kFirstRowWarps)) {
            const uint32_t stride = 32 * apply_warps;
            for (uint32_t u = threadIdx.x - 32 * kFirstRowWarps; u < M.presence.n_updates; u += stride)
                presence_apply(M.presence, M.presence.updates + 9ull * u);
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicAdd(&applied_warps, 1u);
            return;
        }
    }
    const uint32_t c = blockIdx.x * kFirstRowWarps + wid;
    if (c >= n_chains) return;
    FirstRowSmem& s = smem[wid];
    // one chain: its row-0 tokens came in the kernel parameters (no PCIe
    // round trips for the descriptor and the tokens); else mapped memory
    const bool inl = one.n != ~0u;
    ChainDesc cd;
    if (!inl) cd = chains[c];
    const uint32_t n = inl ? one.n : min(P.chunk_size, cd.n_tokens);
    uint32_t flag = 1;  // done, absent
    uint32_t h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool row_was_hit = false;
    uint64_t row_key = 0;
    if (n > 0) {
        // stage the row's tokens and its fingerprint (memo_fingerprint_kernel's)
        uint64_t fp = 0;
        for (uint32_t i = lane; i < n; i += 32) {
            const uint32_t t = inl ? one.tok[i] : tokens[cd.token_off + i];
            s.tok[i] = t;
            fp ^= mix64((uint64_t(t) << 32) | i);
        }
        if (lane == 0) s.tok[n] = 0;
        if (lane < 8)
            s.parent[lane] = (uint32_t(cd.parent[4 * lane]) << 24) | (uint32_t(cd.parent[4 * lane + 1]) << 16) |
                             (uint32_t(cd.parent[4 * lane + 2]) << 8) | uint32_t(cd.parent[4 * lane + 3]);
#pragma unroll
        for (int o = 16; o; o >>= 1) fp ^= __shfl_xor_sync(0xffffffffu, fp, o);
        __syncwarp();
        if (trace != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_staged));
        const uint64_t row_fp = mix64(fp ^ (uint64_t(n) * 0xc2b2ae3d27d4eb4full));  // k = 0
        const uint64_t key = mix64(row_fp ^ parent_fingerprint(cd.parent));
        row_key = key;
        // memo probe + exact verification of a hit (memo_verify_kernel's check)
        uint32_t d[8], ent = kNoEntry;
        bool hit = false;
        if (M.slots != nullptr) {
            if (lane == 0) hit = memo_probe(M, key, d, &ent);
            hit = __shfl_sync(0xffffffffu, hit, 0);
            if (hit) {
                ent = __shfl_sync(0xffffffffu, ent, 0);
#pragma unroll
                for (int i = 0; i < 8; ++i) d[i] = __shfl_sync(0xffffffffu, d[i], 0);
                const uint32_t* e = M.entries + uint64_t(ent) * M.entry_words;
                uint32_t dl = 0;  // d[lane] without a dynamically indexed (local-memory) array
#pragma unroll
                for (int i = 0; i < 8; ++i) dl = lane == uint32_t(i) ? d[i] : dl;
                uint32_t bad = 0;
                if (lane < 8) bad |= (e[lane] ^ s.parent[lane]) | (e[8 + lane] ^ dl);
                if (lane == 0) bad |= e[16] ^ n;
                for (uint32_t i = lane; i < n; i += 32) bad |= e[17 + i] ^ s.tok[i];
                hit = !__any_sync(0xffffffffu, bad != 0);
            }
        }
        if (M.stats != nullptr && lane == 0) atomicAdd(M.stats + (hit ? 0 : 1), 1ull);
        row_was_hit = hit;
        // the pending presence changes (and the witness) are applied from here on
        if (lane == 0 && apply_warps != 0) {
            while (atomicAdd(&applied_warps, 0u) < apply_warps) {
            }
            __threadfence();
        }
        __syncwarp();
        bool witnessed_absent = false;
        if (!hit && M.presence.slots != nullptr) {
            if (lane == 0) {
                witnessed_absent = !witness_may_hold(M.presence, key);
                if (witnessed_absent && M.stats != nullptr) atomicAdd(M.stats + 2, 1ull);
            }
            witnessed_absent = __shfl_sync(0xffffffffu, witnessed_absent, 0);
        }
        if (witnessed_absent) {
            flag |= 4u;  // absent, digest not computed
        } else if (hit) {
#pragma unroll
            for (int i = 0; i < 8; ++i) h[i] = d[i];
        } else {
            // SHA-256 of the chunk: words and schedules lane-parallel, rounds serial
            const uint32_t hdr = 2 + P.tag_len + 32;
            const uint32_t len = hdr + 4 * n;
            const uint32_t nblocks = (len + 9 + 63) / 64;
            const uint32_t end = 64 * nblocks;
            for (uint32_t jw = lane; jw < 16 * nblocks; jw += 32)
                s.w[jw] = pair_msg_word(s.tok, s.parent, P, hdr, len, end, jw);
            __syncwarp();
            for (uint32_t blk = lane; blk < nblocks; blk += 32) expand_block(s.w + 16 * blk, s.kw + 64 * blk);
            __syncwarp();
            uint32_t st[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                              0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
#pragma unroll 1
            for (uint32_t blk = 0; blk < nblocks; ++blk) compress_kw(st, s.kw + 64 * blk);
#pragma unroll
            for (int i = 0; i < 8; ++i) h[i] = st[i];
        }
        if (trace != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_hashed));
        if (lane == 0 && M.presence.slots != nullptr && !witnessed_absent && presence_has(M.presence, h)) flag |= 2u;
    }
    uint32_t hl = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) hl = lane == uint32_t(i) ? h[i] : hl;
    if (lane < 8) digests_out[8 * c + lane] = __byte_perm(hl, 0, 0x0123);
    __syncwarp();
    if (lane == 0 && trace != nullptr) {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        trace[4 * c] = t_start;
        trace[4 * c + 1] = t_staged;
        trace[4 * c + 2] = t_hashed;
        trace[4 * c + 3] = t_end;
    }
    if (lane == 0) {  // the result first (the host is spinning on it) ...
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags_out + c), "r"(flag) : "memory");
    }
    // ... then the memo link of a hashed row (the host syncs the stream
    // before the next launch reads the memo)
    if (n > 0 && M.slots != nullptr && !row_was_hit && !(flag & 4u)) memo_insert(M, s.parent, s.tok, n, row_key, lane, h);
}

// The pending presence changes alone (one thread each), before a lookup.
__global__ void presence_apply_kernel(const PresenceView P) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < P.n_updates; u += gridDim.x * blockDim.x)
        presence_apply(P, P.updates + 9ull * u);
}

// Test hook: corrupt the digest carried by every published slot, so every
// optimistic memo hit must be caught by memo_verify_kernel.
__global__ void memo_poison_kernel(unsigned long long* slots, uint32_t n_slots) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_slots; i += gridDim.x * blockDim.x) {
        unsigned long long* sp = slots + 8ull * i;
        if (*sp != 0 && *sp != kBusy) sp[2] ^= 0x1ull;
    }
}

// Plain SHA-256 of a short byte string (model_tag_hash, src/hash.cpp:41-44):
// one thread, message bytes read from (mapped) memory.
__global__ void sha256_bytes_kernel(const uint8_t* __restrict__ data, uint32_t n,
                                    uint8_t* __restrict__ out) {
    uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                     0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    const uint32_t nblocks = (n + 9 + 63) / 64;
    const uint32_t end = 64 * nblocks;
    for (uint32_t b = 0; b < nblocks; ++b) {
        uint32_t w[16];
        for (int i = 0; i < 16; ++i) {
            uint32_t word = 0;
            for (int k = 0; k < 4; ++k) {
                const uint32_t o = 64 * b + 4 * i + k;
                uint32_t byte;
                if (o < n) byte = data[o];
                else if (o == n) byte = 0x80;
                else if (o >= end - 8) byte = uint32_t((uint64_t(n) * 8) >> (8 * (end - 1 - o))) & 0xff;
                else byte = 0;
                word = (word << 8) | byte;
            }
            w[i] = word;
        }
        compress(h, w);
    }
    for (int i = 0; i < 8; ++i)
        for (int k = 0; k < 4; ++k) out[4 * i + k] = uint8_t(h[i] >> (24 - 8 * k));
}

}  // namespace

cudaError_t launch_memo_stage(const uint32_t* src, uint32_t* dst, const ChainDesc* chains, uint32_t n_chains,
                              uint32_t total_rows, const HashParams& params, const MemoView& memo,
                              cudaStream_t s, const unsigned long long* chain_src) {
    if (total_rows == 0) return cudaSuccess;
    note_launch();
    const uint32_t blocks = (total_rows * 32 + 127) / 128;
    memo_fingerprint_kernel<<<blocks, 128, 0, s>>>(src, dst, chains, n_chains, total_rows, params, memo, nullptr,
                                                    chain_src);
    return cudaGetLastError();
}

cudaError_t launch_memo_stage_chains(const uint32_t* src, uint32_t* dst, const ChainDesc* chains_host,
                                     ChainDesc* chains_dev, uint32_t n_chains, uint32_t total_rows,
                                     const HashParams& params, const MemoView& memo, cudaStream_t s,
                                     const unsigned long long* chain_src) {
    if (n_chains > kStageChains) {  // too many to stage per block: copy them first
        cudaError_t e = launch_sm_copy(chains_host, chains_dev, n_chains * sizeof(ChainDesc), s);
        if (e != cudaSuccess) return e;
        return launch_memo_stage(src, dst, chains_dev, n_chains, total_rows, params, memo, s, chain_src);
    }
    if (total_rows == 0) return launch_sm_copy(chains_host, chains_dev, n_chains * sizeof(ChainDesc), s);
    note_launch();
    const uint32_t blocks = (total_rows * 32 + 127) / 128;
    memo_fingerprint_kernel<<<blocks, 128, 0, s>>>(src, dst, chains_host, n_chains, total_rows, params, memo,
                                                    chains_dev, chain_src);
    return cudaGetLastError();
}

cudaError_t launch_first_row(const uint32_t* tokens, const ChainDesc* chains, uint32_t n_chains,
                             const HashParams& params, const MemoView& memo, uint32_t* digests_out,
                             uint32_t* flags_out, cudaStream_t s, unsigned long long* trace,
                             const FirstRowInline* one) {
    if (n_chains == 0) return cudaSuccess;
    if (params.chunk_size > uint32_t(kWarpChunkMax)) return cudaErrorInvalidValue;
    note_launch();
    const uint32_t blocks = (n_chains + kFirstRowWarps - 1) / kFirstRowWarps;
    FirstRowInline none;
    none.n = ~0u;
    uint32_t threads = 32 * kFirstRowWarps;
    if (blocks == 1 && memo.presence.n_updates != 0)  // + warps applying the presence changes
        threads += std::min<uint32_t>(kFirstRowMaxThreads - 32 * kFirstRowWarps, (memo.presence.n_updates + 31) / 32 * 32);
    first_row_kernel<<<blocks, threads, 0, s>>>(tokens, chains, n_chains, params, memo, digests_out,
                                                             flags_out, trace, one ? *one : none);
    return cudaGetLastError();
}

cudaError_t launch_presence_apply(const PresenceView& v, cudaStream_t s) {
    if (v.n_updates == 0 || v.slots == nullptr) return cudaSuccess;
    note_launch();
    const uint32_t blocks = std::min<uint32_t>((v.n_updates + 255) / 256, 148);
    presence_apply_kernel<<<blocks, 256, 0, s>>>(v);
    return cudaGetLastError();
}

cudaError_t launch_memo_probe(const ChainDesc* chains, uint32_t n_chains, const HashParams& params,
                              uint8_t* out, const MemoView& memo, cudaStream_t s) {
    if (n_chains == 0 || !memo.slots || !memo.first_miss) return cudaSuccess;
    note_launch();
    memo_probe_kernel<<<n_chains, kProbeThreads, 0, s>>>(chains, params, out, memo);
    return cudaGetLastError();
}

cudaError_t launch_memo_verify(const uint32_t* tokens, const ChainDesc* chains, uint32_t n_chains,
                               uint32_t total_rows, const HashParams& params, const uint8_t* dev_out,
                               const MemoView* memo, uint8_t* out, unsigned int* first_bad,
                               cudaStream_t s) {
    if (total_rows == 0) return cudaSuccess;
    note_launch();
    MemoView m;
    if (memo) m = *memo;
    const uint32_t blocks = (total_rows * 32 + 127) / 128;
    memo_verify_kernel<<<blocks, 128, 0, s>>>(tokens, chains, n_chains, total_rows, params, dev_out, m,
                                              out, first_bad);
    return cudaGetLastError();
}

cudaError_t launch_memo_poison(const MemoView& m, cudaStream_t s) {
    if (!m.slots) return cudaSuccess;
    note_launch();
    memo_poison_kernel<<<148, 256, 0, s>>>(m.slots, m.slot_mask + 1);
    return cudaGetLastError();
}

cudaError_t launch_sha256_bytes(const uint8_t* data, uint32_t n, uint8_t* out, cudaStream_t s) {
    note_launch();
    sha256_bytes_kernel<<<1, 1, 0, s>>>(data, n, out);
    return cudaGetLastError();
}

cudaError_t launch_hash_chains(const uint32_t* tokens, const ChainDesc* chains, uint32_t n_chains,
                               const HashParams& params, uint8_t* out, cudaStream_t stream,
                               const MemoView* memo) {
    if (n_chains == 0) return cudaSuccess;
    if (params.tag_len > uint32_t(kMaxTagBytes) || params.chunk_size == 0)
        return cudaErrorInvalidValue;
    note_launch();
    if (params.chunk_size <= uint32_t(kWarpChunkMax)) {
        MemoView m;
        if (memo) m.max_rows = memo->max_rows;
        if (memo && memo->slots && memo->entry_words == 17 + params.chunk_size) {
            m = *memo;
            if (m.first_miss != nullptr) {
                memo_probe_kernel<<<n_chains, kProbeThreads, 0, stream>>>(chains, params, out, m);
                note_launch();
            }
        }
        const int pblocks = int((n_chains + kPairsPerCta - 1) / kPairsPerCta);
        hash_chains_pair_kernel<<<pblocks, 64 * kPairsPerCta, 0, stream>>>(tokens, chains, n_chains, params,
                                                                         out, m);
    } else {
        const int threads = 128;
        const int blocks = int((n_chains + threads - 1) / threads);
        hash_chains_kernel<<<blocks, threads, 0, stream>>>(tokens, chains, n_chains, params, out);
    }
    return cudaGetLastError();
}

}  // namespace tkv
