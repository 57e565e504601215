// K4 — synthetic KV on the device, bit-exact with synth_token_kv
// (src/synth.cpp:7-20): the 8-byte word at byte offset i of the row for
// (token, layer, position) is splitmix64(base + i) stored little-endian, with
// base = splitmix64(seed ^ token<<32 ^ layer<<16 ^ splitmix64(position)) and
// seed = fnv1a64(model_tag) (synth.hpp:27-30).
//
// This is the engine's "compute" stand-in (SimEngine::write_tokens,
// src/sim_engine.cpp:43-64): it fills pages in place so parity and the bench
// run at full scale without shipping inputs over PCIe. verify_pages is the
// device-side byte oracle used for the full-size property checks
// (SimEngine::verify_loaded, src/sim_engine.cpp:66-81).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace tkv {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t row_base(uint64_t seed, uint32_t tok, uint32_t layer,
                                             uint64_t pos) {
    return splitmix64(seed ^ (uint64_t(tok) << 32) ^ (uint64_t(layer) << 16) ^ splitmix64(pos));
}

// Address of byte i of the paged row (layer, pos) under layout L.
__device__ __forceinline__ uint8_t* row_byte(const PagedLayout& L, const SynthArgs& A,
                                             uint32_t layer, uint32_t pos, uint32_t i) {
    const uint32_t page_idx = pos / L.page_tokens;
    const uint32_t in_page = pos - page_idx * L.page_tokens;
    const int32_t pid =
        A.table[uint64_t(L.shared_table ? 0 : layer) * A.table_stride + page_idx];
    const uint64_t base = L.layer_base ? L.layer_base[layer] : L.base;
    const uint32_t q = i / L.plane_bytes;
    const uint32_t c = i - q * L.plane_bytes;
    return reinterpret_cast<uint8_t*>(base + uint64_t(uint32_t(pid)) * L.page_stride +
                                      q * L.plane_stride + uint64_t(in_page) * L.token_stride + c);
}

template <bool VERIFY>
__global__ void synth_pages_kernel(const PagedLayout L, const SynthArgs A,
                                   unsigned long long* mismatches) {
    const uint32_t wpr = (L.bpt + 7) / 8;
    const uint32_t ntok = A.pos_end - A.pos_begin;
    const uint64_t total = uint64_t(A.layer_end - A.layer_begin) * ntok * wpr;
    const bool aligned8 = (L.plane_bytes % 8 == 0) && (L.token_stride % 8 == 0) &&
                          (L.page_stride % 8 == 0) && (L.plane_stride % 8 == 0);
    unsigned long long bad = 0;
    for (uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t row = idx / wpr;
        const uint32_t w = uint32_t(idx - row * wpr);
        const uint32_t layer = A.layer_begin + uint32_t(row / ntok);
        const uint32_t pos = A.pos_begin + uint32_t(row % ntok);
        const uint64_t word = splitmix64(row_base(A.seed, A.tokens[pos], layer, pos) + A.row_offset + 8ull * w);
        const uint32_t i0 = 8 * w;
        const uint32_t nb = min(8u, L.bpt - i0);
        if (aligned8 && nb == 8) {
            uint64_t* p = reinterpret_cast<uint64_t*>(row_byte(L, A, layer, pos, i0));
            if constexpr (VERIFY) {
                bad += (*p != word);
            } else {
                *p = word;
            }
        } else {
            uint32_t diff = 0;
            for (uint32_t b = 0; b < nb; ++b) {
                uint8_t* p = row_byte(L, A, layer, pos, i0 + b);
                const uint8_t v = uint8_t(word >> (8 * b));
                if constexpr (VERIFY) {
                    diff |= (*p != v);
                } else {
                    *p = v;
                }
            }
            bad += diff;
        }
    }
    if constexpr (VERIFY) {
        if (bad) atomicAdd(mismatches, bad);
    }
}

// Fast path (16-byte aligned rows, one plane or plane_bytes % 16 == 0): one
// warp per (layer, position) row computes the row base once and writes or
// checks two words per lane per step with 16-byte accesses.
template <bool VERIFY>
__global__ void __launch_bounds__(256)
synth_rows_kernel(const PagedLayout L, const SynthArgs A, unsigned long long* mismatches) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t ntok = A.pos_end - A.pos_begin;
    const uint64_t rows = uint64_t(A.layer_end - A.layer_begin) * ntok;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const uint32_t pairs = L.bpt / 16;
    unsigned long long bad = 0;
    for (uint64_t row = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < rows;
         row += warps) {
        const uint32_t layer = A.layer_begin + uint32_t(row / ntok);
        const uint32_t pos = A.pos_begin + uint32_t(row % ntok);
        const uint64_t base = row_base(A.seed, A.tokens[pos], layer, pos) + A.row_offset;
        for (uint32_t p = lane; p < pairs; p += 32) {
            const uint32_t i0 = 16 * p;
            const uint64_t w0 = splitmix64(base + i0), w1 = splitmix64(base + i0 + 8);
            ulonglong2* dst = reinterpret_cast<ulonglong2*>(row_byte(L, A, layer, pos, i0));
            if constexpr (VERIFY) {
                const ulonglong2 v = *dst;
                bad += (v.x != w0) + (v.y != w1);
            } else {
                *dst = make_ulonglong2(w0, w1);
            }
        }
    }
    if constexpr (VERIFY) {
        if (bad) atomicAdd(mismatches, bad);
    }
}

bool rows_fast(const PagedLayout& L) {
    return L.bpt % 16 == 0 && L.plane_bytes % 16 == 0 && L.token_stride % 16 == 0 &&
           L.page_stride % 16 == 0 && L.plane_stride % 16 == 0 && L.base % 16 == 0;
}

__global__ void synth_chunk_kernel(const uint32_t* __restrict__ tokens, uint64_t seed,
                                   uint32_t start, uint32_t n, uint32_t n_layers, uint32_t bpt,
                                   uint8_t* __restrict__ out) {
    const uint32_t wpr = (bpt + 7) / 8;
    const uint64_t total = uint64_t(n_layers) * n * wpr;
    for (uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t row = idx / wpr;  // row = layer * n + t
        const uint32_t w = uint32_t(idx - row * wpr);
        const uint32_t layer = uint32_t(row / n);
        const uint32_t t = uint32_t(row % n);
        const uint64_t word =
            splitmix64(row_base(seed, tokens[start + t], layer, start + t) + 8ull * w);
        uint8_t* p = out + row * bpt + 8ull * w;
        const uint32_t nb = min(8u, bpt - 8 * w);
        if (nb == 8 && (bpt % 8 == 0)) {
            *reinterpret_cast<uint64_t*>(p) = word;
        } else {
            for (uint32_t b = 0; b < nb; ++b) p[b] = uint8_t(word >> (8 * b));
        }
    }
}

// Checks a chunk payload [n_layers][n][bpt] (e.g. a pinned tier slot read
// over PCIe) against synth; row_offset = this TP shard's byte offset in the
// full row. One warp per (layer, token) row, 8-byte words.
__global__ void __launch_bounds__(256)
verify_chunk_kernel(const uint32_t* __restrict__ tokens, uint64_t seed, uint32_t start, uint32_t n,
                    uint32_t n_layers, uint32_t bpt, uint64_t row_offset, const uint8_t* __restrict__ chunk,
                    unsigned long long* mismatches) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t rows = uint64_t(n_layers) * n;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const uint32_t wpr = (bpt + 7) / 8;
    unsigned long long bad = 0;
    for (uint64_t row = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < rows; row += warps) {
        const uint32_t layer = uint32_t(row / n);
        const uint32_t t = uint32_t(row - uint64_t(layer) * n);
        const uint64_t base = row_base(seed, tokens[start + t], layer, start + t) + row_offset;
        const uint8_t* r = chunk + row * bpt;
        for (uint32_t w = lane; w < wpr; w += 32) {
            const uint64_t word = splitmix64(base + 8ull * w);
            const uint32_t nb = min(8u, bpt - 8 * w);
            uint32_t diff = 0;
            if (nb == 8 && bpt % 8 == 0) {
                diff = *reinterpret_cast<const uint64_t*>(r + 8ull * w) != word;
            } else {
                for (uint32_t b = 0; b < nb; ++b) diff |= r[8 * w + b] != uint8_t(word >> (8 * b));
            }
            bad += diff;
        }
    }
    if (bad) atomicAdd(mismatches, bad);
}

int grid_for(uint64_t total) {
    uint64_t g = (total + 255) / 256;
    return int(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}

}  // namespace

cudaError_t launch_synth_pages(const PagedLayout& L, const SynthArgs& A, cudaStream_t s) {
    if (A.pos_end <= A.pos_begin || A.layer_end <= A.layer_begin) return cudaSuccess;
    const uint64_t total =
        uint64_t(A.layer_end - A.layer_begin) * (A.pos_end - A.pos_begin) * ((L.bpt + 7) / 8);
    note_launch();
    if (rows_fast(L)) {
        const uint64_t rows = uint64_t(A.layer_end - A.layer_begin) * (A.pos_end - A.pos_begin);
        synth_rows_kernel<false><<<grid_for(rows * 32), 256, 0, s>>>(L, A, nullptr);
    } else {
        synth_pages_kernel<false><<<grid_for(total), 256, 0, s>>>(L, A, nullptr);
    }
    return cudaGetLastError();
}

cudaError_t launch_verify_pages(const PagedLayout& L, const SynthArgs& A,
                                unsigned long long* mismatches, cudaStream_t s) {
    if (A.pos_end <= A.pos_begin || A.layer_end <= A.layer_begin) return cudaSuccess;
    const uint64_t total =
        uint64_t(A.layer_end - A.layer_begin) * (A.pos_end - A.pos_begin) * ((L.bpt + 7) / 8);
    note_launch();
    if (rows_fast(L)) {
        const uint64_t rows = uint64_t(A.layer_end - A.layer_begin) * (A.pos_end - A.pos_begin);
        synth_rows_kernel<true><<<grid_for(rows * 32), 256, 0, s>>>(L, A, mismatches);
    } else {
        synth_pages_kernel<true><<<grid_for(total), 256, 0, s>>>(L, A, mismatches);
    }
    return cudaGetLastError();
}

cudaError_t launch_verify_chunk(const uint32_t* tokens, uint64_t seed, uint32_t start, uint32_t n,
                                uint32_t n_layers, uint32_t bpt, uint64_t row_offset, const uint8_t* chunk,
                                unsigned long long* mismatches, cudaStream_t s) {
    if (n == 0 || n_layers == 0) return cudaSuccess;
    note_launch();
    verify_chunk_kernel<<<grid_for(uint64_t(n_layers) * n * 32), 256, 0, s>>>(tokens, seed, start, n, n_layers,
                                                                             bpt, row_offset, chunk, mismatches);
    return cudaGetLastError();
}

cudaError_t launch_synth_chunk(const uint32_t* tokens, uint64_t seed, uint32_t start, uint32_t n,
                               uint32_t n_layers, uint32_t bpt, uint8_t* out, cudaStream_t s) {
    if (n == 0 || n_layers == 0) return cudaSuccess;
    const uint64_t total = uint64_t(n_layers) * n * ((bpt + 7) / 8);
    note_launch();
    synth_chunk_kernel<<<grid_for(total), 256, 0, s>>>(tokens, seed, start, n, n_layers, bpt, out);
    return cudaGetLastError();
}

}  // namespace tkv
