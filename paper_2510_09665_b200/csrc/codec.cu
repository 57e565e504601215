// q8-scale codec on the device, bit-exact with
// Q8ScaleCodec (src/codec.cpp:27-91):
//   payload = signed 16-bit little-endian lanes (+ a raw odd tail byte)
//   scale   = float(max|lane| / 127.0)            (q8_scale_of, codec.cpp:86-94)
//   encode  = round(double(lane) / double(scale)) clamped to [-127, 127], int8
//   decode  = round(double(q) * double(scale)) clamped to [-32768, 32767]
//   blob    = u32le original_len | f32le scale | int8 lanes | odd tail byte
// round() is round-half-away-from-zero in both C and CUDA, and double
// division / multiplication are IEEE correctly rounded on both sides, so the
// bytes match. One launch covers a batch of chunk payloads. Decode is
// HBM-bound. Encode is ONE cooperative launch (q8_encode_fused_kernel):
// warp-specialised absmax warps stream each item from DRAM once, keeping its
// lines in L2, and quantise warps of the same CTAs re-read it from L2 one
// item behind, so DRAM sees the payload once (ncu: 538 MB read for a 537 MB
// payload) instead of twice. 16 x 32 MiB: 0.177-0.187 ms (0.67-0.71 of the
// one-pass bound) vs 0.237 ms for the two-kernel encode, which batches of
// small or few items keep (launch_q8_encode; TKV_Q8_ENCODE=fused|twopass
// forces one). Earlier single-pass tries — an atomic work queue
// (round 1), a CTA quantising one segment behind its own absmax — lost
// their L2 savings to CTAs alternating DRAM and L2 phases.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "kernels.hpp"

namespace tkv {
namespace {

constexpr int kThreads = 256;
constexpr uint64_t kSeg = 64 * 1024;  // payload bytes per CTA work item
constexpr int kUnroll = 4;            // 16-byte vectors in flight per thread
constexpr uint64_t kStride = 16 * kThreads;

// Grid-stride over (item, segment): per-item max |lane| into maxabs[item].
__global__ void __launch_bounds__(kThreads)
q8_absmax_kernel(const CodecItem* __restrict__ items, const uint32_t* __restrict__ seg_base,
                 uint32_t n_items, uint32_t total_segs, int* __restrict__ maxabs) {
    __shared__ int red[kThreads / 32];
    for (uint32_t seg = blockIdx.x; seg < total_segs; seg += gridDim.x) {
        uint32_t lo = 0, hi = n_items;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (seg_base[mid] <= seg) lo = mid; else hi = mid;
        }
        const CodecItem it = items[lo];
        const uint64_t b0 = uint64_t(seg - seg_base[lo]) * kSeg;
        const uint64_t lanes_end = it.bytes & ~uint64_t(1);
        const uint64_t b1 = min(b0 + kSeg, lanes_end);
        int m = 0;
        if ((reinterpret_cast<uint64_t>(it.src) & 15) == 0) {
            // 16-byte loads, 8 lanes each: per-halfword |lane| (non-saturating,
            // so -32768 -> 0x8000 = 32768 unsigned) folded with unsigned max
            const uint64_t vend = b0 + ((b1 - b0) & ~uint64_t(15));
            uint32_t m2 = 0;
            for (uint64_t b = b0 + 16 * threadIdx.x; b < vend; b += kStride * kUnroll) {
                uint4 v[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
                    v[u] = b + u * kStride < vend ? __ldcs(reinterpret_cast<const uint4*>(it.src + b + u * kStride))
                                                  : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
                    m2 = __vmaxu2(m2, __vmaxu2(__vmaxu2(__vabs2(v[u].x), __vabs2(v[u].y)),
                                               __vmaxu2(__vabs2(v[u].z), __vabs2(v[u].w))));
            }
            m = int(max(m2 & 0xffffu, m2 >> 16));
            for (uint64_t b = vend + 2 * threadIdx.x; b + 2 <= b1; b += 2 * kThreads)
                m = max(m, abs(int32_t(int16_t(uint16_t(it.src[b] | (it.src[b + 1] << 8))))));
        } else {
            for (uint64_t b = b0 + 2 * threadIdx.x; b + 2 <= b1; b += 2 * kThreads)
                m = max(m, abs(int32_t(int16_t(uint16_t(it.src[b] | (it.src[b + 1] << 8))))));
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            int mm = 0;
            for (int i = 0; i < kThreads / 32; ++i) mm = max(mm, red[i]);
            atomicMax(maxabs + lo, mm);
        }
        __syncthreads();
    }
}

// round(double(lane) / double(scale)) without the division (codec.cpp:42-44),
// in two FP64 instructions per lane. scale is a float (24-bit significand M)
// and |lane| <= 32768, so a quotient Q = |lane| / scale that is not exactly
// k + 1/2 lies at least 1/(2M) >= 2^-25 away from every half-integer. With
// inv = 1/scale rounded UP, Q' = |lane| * inv (exact inside the FMA) is in
// [Q, Q + 2^-45]: an exact tie stays on or just above k + 1/2 (rounds away
// from zero, as round() does) and no other quotient crosses a half-integer.
// fma.rz(|lane|, inv, 2^45 + 1/2) then holds floor(Q' + 1/2) in its integer
// part (round-toward-zero onto the 2^-7 grid of [2^45, 2^46) cannot cross an
// integer), i.e. bits 7.. of the low word. |lane| -> double is the exact 2^52
// magic subtraction (no conversion on the XU pipe). (The reference's
// correctly rounded double quotient rounds the same way for the same reason.)
__device__ __forceinline__ uint32_t quant(int32_t lane, double inv_up) {
    constexpr double kMagic = 4503599627370496.0;  // 2^52
    const double al = __hiloint2double(0x43300000, abs(lane)) - kMagic;  // exact, |lane| <= 32768
    const double t = __fma_rz(al, inv_up, 35184372088832.5);               // 2^45 + 1/2
    const uint32_t q = min(uint32_t(__double2loint(t)) >> 7, 127u);
    return (lane < 0 ? 0u - q : q) & 0xffu;
}

// Four lanes (two little-endian words) -> four q8 bytes, the vector path of
// both encodes, with no magnitude / sign handling. With inv
// STRICTLY above 1/scale (rounded up, bumped one ulp when the reciprocal is
// exact), Q' = lane * inv sits within (0, 2^-44] of Q = lane / scale on the
// side away from zero, so floor(Q' + 1/2) is round-half-away(Q) for either
// sign: a tie +-(k + 1/2) lands just outside it, and non-ties are >= 2^-25
// from every half-integer. The lane enters as the exact double
// (2^52 + (lane + 2^15)) - (2^52 + 2^15) (the bias is the XOR of the sign
// bit), then fma.rz(lane, inv, 2^44 + 2^43 + 1/2) keeps floor(Q' + 1/2) +
// 2^44 + 2^43 on the 2^-8 grid of [2^44, 2^45) for |q| <= 128, so byte 1 of
// its low word is q's int8 bit pattern (2^44 + 2^43 is a multiple of 256).
__device__ __forceinline__ uint32_t quant4s(uint32_t w0, uint32_t w1, double inv) {
    constexpr double kBias = 4503599627403264.0;  // 2^52 + 2^15
    const uint32_t b0 = w0 ^ 0x80008000u, b1 = w1 ^ 0x80008000u;  // lane + 2^15 per halfword
    const uint32_t u[4] = {b0 & 0xffffu, b0 >> 16, b1 & 0xffffu, b1 >> 16};
    uint32_t t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double x = __hiloint2double(0x43300000, int(u[k])) - kBias;  // exact
        t[k] = uint32_t(__double2loint(__fma_rz(x, inv, 26388279066624.5)));  // 2^44 + 2^43 + 1/2
    }
    return __byte_perm(__byte_perm(t[0], t[1], 0x0051), __byte_perm(t[2], t[3], 0x0051), 0x5410);
}

// 1/scale rounded up, and strictly above 1/scale (quant4s' tie argument)
__device__ __forceinline__ double inv_strict_up(float scale) {
    if (!(scale > 0.f)) return 0.0;
    const double sc = double(scale);
    double inv = __drcp_ru(sc);
    if (__fma_rn(inv, sc, -1.0) == 0.0) inv = __longlong_as_double(__double_as_longlong(inv) + 1);
    return inv;
}

__device__ __forceinline__ void quant_vectors(const uint8_t* __restrict__ src, uint8_t* __restrict__ out,
                                              uint64_t b0, uint64_t vend, double inv) {
    for (uint64_t b = b0 + 16 * threadIdx.x; b < vend; b += kStride * kUnroll) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (b + u * kStride < vend) v[u] = __ldcs(reinterpret_cast<const uint4*>(src + b + u * kStride));
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (b + u * kStride >= vend) break;
            __stcs(reinterpret_cast<uint2*>(out + (b + u * kStride) / 2),
                   make_uint2(quant4s(v[u].x, v[u].y, inv), quant4s(v[u].z, v[u].w, inv)));
        }
    }
}

__global__ void __launch_bounds__(kThreads)
q8_encode_kernel(const CodecItem* __restrict__ items, const uint32_t* __restrict__ seg_base,
                 uint32_t n_items, uint32_t total_segs, const int* __restrict__ maxabs) {
    for (uint32_t seg = blockIdx.x; seg < total_segs; seg += gridDim.x) {
        uint32_t lo = 0, hi = n_items;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (seg_base[mid] <= seg) lo = mid; else hi = mid;
        }
        const CodecItem it = items[lo];
        const float scale = float(double(maxabs[lo]) / 127.0);
        const double inv = inv_strict_up(scale);  // scale 0: every lane is 0
        const uint32_t local = seg - seg_base[lo];
        if (local == 0 && threadIdx.x == 0) {
            const uint32_t len = uint32_t(it.bytes);
            uint32_t sb;
            memcpy(&sb, &scale, 4);
            for (int i = 0; i < 4; ++i) {
                it.dst[i] = uint8_t(len >> (8 * i));
                it.dst[4 + i] = uint8_t(sb >> (8 * i));
            }
            if (it.bytes & 1) it.dst[8 + it.bytes / 2] = it.src[it.bytes - 1];  // raw odd tail
        }
        const uint64_t b0 = uint64_t(local) * kSeg;
        const uint64_t lanes_end = it.bytes & ~uint64_t(1);
        const uint64_t b1 = min(b0 + kSeg, lanes_end);
        uint8_t* out = it.dst + 8;
        uint64_t vend = b0;
        if (((reinterpret_cast<uint64_t>(it.src) & 15) | (reinterpret_cast<uint64_t>(out) & 7)) == 0) {
            vend = b0 + ((b1 - b0) & ~uint64_t(15));
            quant_vectors(it.src, out, b0, vend, inv);
        }
        for (uint64_t b = vend + 2 * threadIdx.x; b + 2 <= b1; b += 2 * kThreads) {
            const int32_t lane = int32_t(int16_t(uint16_t(it.src[b] | (it.src[b + 1] << 8))));
            out[b / 2] = uint8_t(quant(lane, inv));
        }
    }
}

// ---- single-pass encode: warp-specialised, item-pipelined persistent grid ---
//
// The scale is one per item (the whole chunk payload), so no byte can be
// quantised before the item's absmax is complete, and the two-kernel encode
// reads every payload twice from DRAM. Here one cooperative grid (one CTA
// per SM, all resident) splits each CTA's warps into two roles:
//   * absmax warps stream item p from DRAM with 256-bit loads that keep
//     their lines in L2 (L2::evict_last), 8 loads in flight per lane, and
//     count the CTA in on item p's arrival counter when done;
//   * quantise warps wait until every CTA arrived for item q (normally
//     already true: the absmax warps run one item ahead), then re-read item
//     q from L2 as a last use (L2::evict_first), quantise and stream the
//     int8 lanes out, and count the CTA in on item q's done counter.
// The absmax warps start item p only once item p - 2 is quantised
// everywhere, so L2 holds at most the item being quantised and the one
// being streamed (2 x 32 MiB chunk payloads of the 8B model in 126 MB).
// DRAM then sees the payload once plus the int8 output (the 1.5 P of the
// single-pass bound) and both roles run concurrently: the DRAM stream does
// not stop while lanes are quantised. Roles synchronise with named barriers
// (never __syncthreads) and per-item global counters, so there is no
// grid-wide barrier. Tile -> CTA assignment rotates per item.
constexpr int kFusedThreads = 1024;
constexpr uint32_t kCounterStride = 32;  // unsigned per counter: one 128-byte line each
constexpr int kBarA = 1, kBarB = 2;               // named barriers (0 = __syncthreads)

struct V32 {
    uint32_t w[8];
};
// 256-bit loads (sm_100) carrying an L2 eviction priority
__device__ __forceinline__ V32 ld_keep_l2(const uint8_t* p) {
    V32 v;
    asm volatile("ld.global.L1::no_allocate.L2::evict_last.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]),
                   "=r"(v.w[6]), "=r"(v.w[7])
                 : "l"(p));
    return v;
}
__device__ __forceinline__ V32 ld_last_use(const uint8_t* p) {
    V32 v;
    asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]),
                   "=r"(v.w[6]), "=r"(v.w[7])
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void bar_named(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void await_count(const unsigned* p, unsigned want) {
    while (ld_acquire_u32(p) < want) __nanosleep(100);
}
__device__ __forceinline__ int lane_at(const uint8_t* p, uint64_t b) {
    return int32_t(int16_t(uint16_t(p[b] | (p[b + 1] << 8))));
}

template <int kBThreads, int kBUnroll>
__device__ __forceinline__ void quant_tiles(const uint8_t* __restrict__ src, uint8_t* __restrict__ out,
                                            uint64_t vend, uint32_t first, uint32_t ntiles, uint32_t bt,
                                            double inv) {
    constexpr uint64_t kStrideB = 32ull * kBThreads;
    constexpr uint64_t kBTile = kStrideB * kBUnroll;
    for (uint32_t t = first; t < ntiles; t += gridDim.x) {
        const uint64_t b = uint64_t(t) * kBTile + 32 * bt;
        V32 v[kBUnroll];
#pragma unroll
        for (int u = 0; u < kBUnroll; ++u)
            if (b + u * kStrideB < vend) v[u] = ld_last_use(src + b + u * kStrideB);
#pragma unroll
        for (int u = 0; u < kBUnroll; ++u) {
            if (b + u * kStrideB >= vend) break;
            uint2* o = reinterpret_cast<uint2*>(out + (b + u * kStrideB) / 2);  // blob lanes are 8-aligned
            __stcs(o, make_uint2(quant4s(v[u].w[0], v[u].w[1], inv), quant4s(v[u].w[2], v[u].w[3], inv)));
            __stcs(o + 1, make_uint2(quant4s(v[u].w[4], v[u].w[5], inv), quant4s(v[u].w[6], v[u].w[7], inv)));
        }
    }
}

template <int kFThreads, int kAWarps, int kAUnroll, int kBUnroll, int kAhead = 1>
__global__ void __launch_bounds__(kFThreads, 1)
q8_encode_fused_kernel(const CodecItem* __restrict__ items, uint32_t n_items, int* __restrict__ maxabs,
                       unsigned* __restrict__ arrive, unsigned* __restrict__ done) {
    constexpr int kBWarps = kFThreads / 32 - kAWarps;  // quantise warps per CTA
    constexpr int kAThreads = 32 * kAWarps, kBThreads = 32 * kBWarps;
    constexpr uint64_t kATile = 32ull * kAThreads * kAUnroll;
    constexpr uint64_t kBTile = 32ull * kBThreads * kBUnroll;
    __shared__ int red[2][kAWarps];
    const uint32_t G = gridDim.x;
    auto first_tile = [&](uint32_t item) {  // this CTA's first tile of an item (rotated assignment)
        const uint32_t rot = uint32_t((uint64_t(item) * 2654435761ull) % G);
        return (blockIdx.x + G - rot) % G;
    };
    const uint32_t warp = threadIdx.x >> 5;
    if (warp < kAWarps) {  // ---- absmax role
        const uint32_t at = threadIdx.x;
        const uint64_t gt = uint64_t(blockIdx.x) * kAThreads + at, gn = uint64_t(G) * kAThreads;
        constexpr uint64_t kStrideA = 32ull * kAThreads;
        for (uint32_t p = 0; p < n_items; ++p) {
            if (p >= kAhead + 1) {  // L2 budget: item p - 1 - kAhead quantised everywhere
                if (at == 0) await_count(done + uint64_t(p - 1 - kAhead) * kCounterStride, G);
                bar_named(kBarA, kAThreads);
            }
            const CodecItem it = items[p];
            const uint64_t lanes_end = it.bytes & ~uint64_t(1);
            int m = 0;
            uint64_t vend = 0;
            if ((reinterpret_cast<uint64_t>(it.src) & 31) == 0) {
                vend = lanes_end & ~uint64_t(31);
                const uint32_t ntiles = uint32_t((vend + kATile - 1) / kATile);
                // signed per-halfword max and min (one VIMNMX each per word);
                // max|lane| = max(max, -min) in 32 bits (-(-32768) = 32768)
                uint32_t hi2 = 0, lo2 = 0;
                for (uint32_t t = first_tile(p); t < ntiles; t += G) {
                    const uint64_t b = uint64_t(t) * kATile + 32 * at;
                    V32 v[kAUnroll];
#pragma unroll
                    for (int u = 0; u < kAUnroll; ++u) {
                        if (b + u * kStrideA < vend) v[u] = ld_keep_l2(it.src + b + u * kStrideA);
                        else v[u] = V32{};
                    }
#pragma unroll
                    for (int u = 0; u < kAUnroll; ++u)
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            hi2 = __vmaxs2(hi2, v[u].w[k]);
                            lo2 = __vmins2(lo2, v[u].w[k]);
                        }
                }
                m = max(max(int(int16_t(hi2 & 0xffffu)), int(int16_t(hi2 >> 16))),
                        -min(int(int16_t(lo2 & 0xffffu)), int(int16_t(lo2 >> 16))));
            }
            for (uint64_t b = vend + 2 * gt; b + 2 <= lanes_end; b += 2 * gn)  // unaligned item / tail
                m = max(m, abs(lane_at(it.src, b)));
#pragma unroll
            for (int off = 16; off; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
            if ((at & 31) == 0) red[p & 1][warp] = m;
            bar_named(kBarA, kAThreads);
            if (at == 0) {
                int mm = 0;
                for (int i = 0; i < kAWarps; ++i) mm = max(mm, red[p & 1][i]);
                if (mm) atomicMax(maxabs + p, mm);
                __threadfence();
                atomicAdd(arrive + uint64_t(p) * kCounterStride, 1u);
            }
        }
        return;
    }
    // ---- quantise role
    const uint32_t bt = threadIdx.x - kAThreads;
    const uint64_t gt = uint64_t(blockIdx.x) * kBThreads + bt, gn = uint64_t(G) * kBThreads;
    for (uint32_t q = 0; q < n_items; ++q) {
        if (bt == 0) await_count(arrive + uint64_t(q) * kCounterStride, G);  // item q's absmax complete everywhere
        bar_named(kBarB, kBThreads);
        const CodecItem it = items[q];
        const float scale = float(double(__ldcg(maxabs + q)) / 127.0);
        const double inv = inv_strict_up(scale);  // scale 0: every lane is 0
        if (blockIdx.x == 0 && bt == 0) {
            const uint32_t len = uint32_t(it.bytes);
            uint32_t sb;
            memcpy(&sb, &scale, 4);
            for (int i = 0; i < 4; ++i) {
                it.dst[i] = uint8_t(len >> (8 * i));
                it.dst[4 + i] = uint8_t(sb >> (8 * i));
            }
            if (it.bytes & 1) it.dst[8 + it.bytes / 2] = it.src[it.bytes - 1];  // raw odd tail
        }
        const uint64_t lanes_end = it.bytes & ~uint64_t(1);
        uint8_t* out = it.dst + 8;
        uint64_t vend = 0;
        if (((reinterpret_cast<uint64_t>(it.src) & 31) | (reinterpret_cast<uint64_t>(out) & 7)) == 0) {
            vend = lanes_end & ~uint64_t(31);
            const uint32_t ntiles = uint32_t((vend + kBTile - 1) / kBTile);
            quant_tiles<kBThreads, kBUnroll>(it.src, out, vend, first_tile(q), ntiles, bt, inv);
        }
        for (uint64_t b = vend + 2 * gt; b + 2 <= lanes_end; b += 2 * gn)
            out[b / 2] = uint8_t(quant(lane_at(it.src, b), inv));
        bar_named(kBarB, kBThreads);
        if (bt == 0) {
            __threadfence();
            atomicAdd(done + uint64_t(q) * kCounterStride, 1u);
        }
    }
}

// round(double(q) * double(scale)) clamped to int16 (codec.cpp:62-68), for
// any scale bit pattern the blob carries. The product v of an 8-bit and a
// 24-bit significand is exact; v +- 1/2 is exact too wherever it can matter
// (|v| < 2^15 with no bits below 2^-38 — a scale small enough to have them
// gives |v| < 1/2), so truncating v +- 1/2 rounds half away from zero. The
// truncating conversion saturates +-inf; a NaN product (0 * inf, NaN scale)
// is -32768, as std::max(-32768.0, NaN) returns its first argument.
__device__ __forceinline__ uint32_t dequant(int8_t q, double sc) {
    const double v = double(q) * sc;
    if (v != v) return 0x8000u;
    int32_t r = __double2int_rz(v + (v < 0.0 ? -0.5 : 0.5));
    r = max(-32768, min(32767, r));
    return uint32_t(uint16_t(int16_t(r)));
}

__global__ void __launch_bounds__(kThreads)
q8_decode_kernel(const CodecItem* __restrict__ items, const uint32_t* __restrict__ seg_base,
                 uint32_t n_items, uint32_t total_segs) {
    // An item has one scale, so its 256 possible codes decode through a
    // 256-entry table built per segment: one shared-memory load per lane.
    __shared__ uint16_t table[256];
    for (uint32_t seg = blockIdx.x; seg < total_segs; seg += gridDim.x) {
        uint32_t lo = 0, hi = n_items;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (seg_base[mid] <= seg) lo = mid; else hi = mid;
        }
        const CodecItem it = items[lo];  // src = blob, dst = payload, bytes = original length
        const uint32_t sb = uint32_t(it.src[4]) | (uint32_t(it.src[5]) << 8) |
                            (uint32_t(it.src[6]) << 16) | (uint32_t(it.src[7]) << 24);
        float scale;
        memcpy(&scale, &sb, 4);
        const uint32_t local = seg - seg_base[lo];
        if (local == 0 && threadIdx.x == 0 && (it.bytes & 1))
            it.dst[it.bytes - 1] = it.src[8 + it.bytes / 2];
        const uint64_t b0 = uint64_t(local) * kSeg;
        const uint64_t b1 = min(b0 + kSeg, it.bytes & ~uint64_t(1));
        const double sc = double(scale);
        __syncthreads();  // previous segment done with the table
        for (uint32_t c = threadIdx.x; c < 256; c += kThreads) table[c] = uint16_t(dequant(int8_t(uint8_t(c)), sc));
        __syncthreads();
        uint64_t vend = b0;
        if (((reinterpret_cast<uint64_t>(it.src + 8) & 7) | (reinterpret_cast<uint64_t>(it.dst) & 15)) == 0) {
            vend = b0 + ((b1 - b0) & ~uint64_t(15));
            for (uint64_t b = b0 + 16 * threadIdx.x; b < vend; b += kStride * kUnroll) {
                uint2 qv[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
                    if (b + u * kStride < vend)
                        qv[u] = __ldcs(reinterpret_cast<const uint2*>(it.src + 8 + (b + u * kStride) / 2));
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    if (b + u * kStride >= vend) break;
                    uint32_t o[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t w = k < 2 ? qv[u].x : qv[u].y;
                        o[k] = uint32_t(table[(w >> (16 * (k & 1))) & 0xff]) |
                               (uint32_t(table[(w >> (16 * (k & 1) + 8)) & 0xff]) << 16);
                    }
                    __stcs(reinterpret_cast<uint4*>(it.dst + b + u * kStride), make_uint4(o[0], o[1], o[2], o[3]));
                }
            }
        }
        for (uint64_t b = vend + 2 * threadIdx.x; b + 2 <= b1; b += 2 * kThreads) {
            const uint32_t lane = table[it.src[8 + b / 2]];
            it.dst[b] = uint8_t(lane & 0xff);
            it.dst[b + 1] = uint8_t(lane >> 8);
        }
    }
}

int grid(uint32_t segs) { return int(segs < 148u * 8 ? (segs ? segs : 1) : 148u * 8); }

}  // namespace

uint64_t q8_encode_scratch_bytes(uint32_t n) {
    return ((uint64_t(n) * 4 + 127) & ~uint64_t(127)) + 2ull * n * kCounterStride * 4;
}

uint32_t codec_segments(uint64_t bytes) { return uint32_t((bytes + kSeg - 1) / kSeg) + (bytes == 0); }

namespace {
// Resident grid of the single-pass encode per device (one CTA per SM).
std::mutex g_fused_mu;
std::map<int, int> g_fused_grid;

// TKV_Q8_ENCODE: unset = by batch shape (below), "fused" = the single-pass
// encode for every batch, "twopass" = the two kernels for every batch.
int encode_mode() {
    static const int mode = [] {
        const char* v = std::getenv("TKV_Q8_ENCODE");
        if (v && std::strcmp(v, "twopass") == 0) return 2;
        if (v && std::strcmp(v, "fused") == 0) return 1;
        return 0;
    }();
    return mode;
}
}  // namespace

cudaError_t launch_q8_encode(const CodecItem* items, const uint32_t* seg_base, uint32_t n_items,
                             uint32_t total_segs, int* maxabs, cudaStream_t s) {
    if (n_items == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(maxabs, 0, n_items * sizeof(int), s);
    if (e != cudaSuccess) return e;
    // The single-pass encode saves one DRAM read of each item (P / 6.4 TB/s:
    // ~5 us per 32 MiB) but pays a grid-wide hand-off per item (~4 us) and a
    // pipeline fill of one item: it wins from ~24 MiB items on and with a
    // few items to overlap (16 x 32 MiB: 0.18 vs 0.24 ms; 6 x 80 MiB: 0.197
    // vs 0.221; 64 x 8 MiB: 0.288 vs 0.239; 4 x 10 MiB: 0.032 vs 0.027,
    // profiles/r02_codec.jsonl). Other batches take the two-kernel encode.
    const int mode = encode_mode();
    if (mode == 1 || (mode == 0 && n_items >= 3 && uint64_t(total_segs) >= 384ull * n_items)) {
        // scratch (q8_encode_scratch_bytes): maxabs[n], then one 128-byte
        // line per item for its arrival counter and one for its done counter
        // (spinning warps never share a line with another item's atomics) —
        // in the caller's per-call scratch, so concurrent encodes never share
        // them
        unsigned* arrive = reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(maxabs) +
                                                       ((uint64_t(n_items) * 4 + 127) & ~uint64_t(127)));
        unsigned* done = arrive + uint64_t(n_items) * kCounterStride;
        int dev = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
        int grid = 0;
        {
            std::lock_guard<std::mutex> lk(g_fused_mu);
            int& g = g_fused_grid[dev];
            if (g == 0) {
                int per_sm = 0, sms = 0;
                if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                         &per_sm, q8_encode_fused_kernel<kFusedThreads, 12, 6, 2, 2>, kFusedThreads, 0)) != cudaSuccess)
                    return e;
                if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
                if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
                g = sms;  // one CTA per SM (launch bounds: 1024 threads, 1 per SM)
            }
            grid = g;
        }
        if ((e = cudaMemsetAsync(arrive, 0, 2ull * n_items * kCounterStride * sizeof(unsigned), s)) != cudaSuccess)
            return e;
        void* args[] = {const_cast<CodecItem**>(&items), &n_items, &maxabs, &arrive, &done};
        note_launch();
        // 12 absmax warps x 6 x 32-byte loads in flight, 20 quantise warps x 2,
        // absmax up to two items ahead of the quantise (measured against
        // 4-24 absmax warps, 1-3 items ahead: profiles/r02_codec.jsonl)
        const void* fn = reinterpret_cast<const void*>(q8_encode_fused_kernel<kFusedThreads, 12, 6, 2, 2>);
        return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kFusedThreads), args, 0, s);
    }
    note_launch();
    q8_absmax_kernel<<<grid(total_segs), kThreads, 0, s>>>(items, seg_base, n_items, total_segs, maxabs);
    note_launch();
    q8_encode_kernel<<<grid(total_segs), kThreads, 0, s>>>(items, seg_base, n_items, total_segs, maxabs);
    return cudaGetLastError();
}

cudaError_t launch_q8_decode(const CodecItem* items, const uint32_t* seg_base, uint32_t n_items,
                             uint32_t total_segs, cudaStream_t s) {
    if (n_items == 0) return cudaSuccess;
    note_launch();
    q8_decode_kernel<<<grid(total_segs), kThreads, 0, s>>>(items, seg_base, n_items, total_segs);
    return cudaGetLastError();
}

}  // namespace tkv
