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
// HBM-bound; encode reads the payload twice (absmax, then quantise), both
// passes near DRAM speed (the quantise at one fma.rz per lane, quant4).
// Single-pass variants — an atomic work queue (round 1), a persistent grid
// quantising one round behind its absmax (round 2) — cut DRAM reads to
// 1.05-1.12x payload through L2 reuse but ran slower (0.27-0.37 ms vs 0.25
// for 16 x 32 MiB: each CTA alternates a DRAM-latency phase and an L2 phase
// with little memory parallelism), so the two kernels stay.
#include <cuda_runtime.h>

#include <cstdint>

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
// the encode: |lane| as the low word of the double 2^52 + |lane| (one move
// of the constant high word), then ONE fma.rz per lane:
//   fma.rz(2^52 + |lane|, inv, c),  c = 2^44 + 1/2 - 2^52 inv  (kFold)
// is exactly 2^44 + 1/2 + |lane| inv rounded toward zero onto the 2^-8 grid
// of [2^44, 2^45), so byte 1 of its low word is floor(Q' + 1/2) — quant()'s
// value. c is exact when inv < 1/2 (scale > 2: c is a multiple of inv's ulp
// below 2^53 of them); smaller scales take quant()'s subtraction first
// (!kFold). No clamp: |lane| <= max|lane| = 127 * scale * (1 +- 2^-24), so
// the byte is at most 127. Signs are applied bytewise: prmt's sign-replicate
// mode turns each lane's high byte into a 0x00 / 0xff mask, and for
// n <= 127, ((n ^ 0x7f) + 1) ^ 0x80 = -n mod 256 with no carry between bytes.
template <bool kFold>
__device__ __forceinline__ uint32_t quant4(uint32_t w0, uint32_t w1, double inv, double c) {
    constexpr double kMagic = 4503599627370496.0;  // 2^52
    const uint32_t a0 = __vabs2(w0), a1 = __vabs2(w1);  // -32768 -> 0x8000 (non-saturating)
    const uint32_t mag[4] = {a0 & 0xffffu, a0 >> 16, a1 & 0xffffu, a1 >> 16};
    uint32_t t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double x = __hiloint2double(0x43300000, int(mag[k]));
        t[k] = uint32_t(__double2loint(kFold ? __fma_rz(x, inv, c) : __fma_rz(x - kMagic, inv, 17592186044416.5)));
    }
    const uint32_t n = __byte_perm(__byte_perm(t[0], t[1], 0x0051), __byte_perm(t[2], t[3], 0x0051), 0x5410);
    uint32_t m;  // 0xff where the lane is negative
    asm("prmt.b32 %0, %1, %2, 0xFDB9;" : "=r"(m) : "r"(w0), "r"(w1));
    const uint32_t neg = ((n ^ 0x7f7f7f7fu) + 0x01010101u) ^ 0x80808080u;
    return (neg & m) | (n & ~m);
}

template <bool kFold>
__device__ __forceinline__ void quant_vectors(const uint8_t* __restrict__ src, uint8_t* __restrict__ out,
                                              uint64_t b0, uint64_t vend, double inv, double c) {
    for (uint64_t b = b0 + 16 * threadIdx.x; b < vend; b += kStride * kUnroll) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (b + u * kStride < vend) v[u] = __ldcs(reinterpret_cast<const uint4*>(src + b + u * kStride));
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (b + u * kStride >= vend) break;
            __stcs(reinterpret_cast<uint2*>(out + (b + u * kStride) / 2),
                   make_uint2(quant4<kFold>(v[u].x, v[u].y, inv, c), quant4<kFold>(v[u].z, v[u].w, inv, c)));
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
        const double inv = scale > 0.f ? __drcp_ru(double(scale)) : 0.0;  // scale 0: every lane is 0
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
            if (inv < 0.5)  // (uniform per item)
                quant_vectors<true>(it.src, out, b0, vend, inv, 17592186044416.5 - inv * 4503599627370496.0);
            else
                quant_vectors<false>(it.src, out, b0, vend, inv, 0.0);
        }
        for (uint64_t b = vend + 2 * threadIdx.x; b + 2 <= b1; b += 2 * kThreads) {
            const int32_t lane = int32_t(int16_t(uint16_t(it.src[b] | (it.src[b + 1] << 8))));
            out[b / 2] = uint8_t(quant(lane, inv));
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

uint32_t codec_segments(uint64_t bytes) { return uint32_t((bytes + kSeg - 1) / kSeg) + (bytes == 0); }

cudaError_t launch_q8_encode(const CodecItem* items, const uint32_t* seg_base, uint32_t n_items,
                             uint32_t total_segs, int* maxabs, cudaStream_t s) {
    if (n_items == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(maxabs, 0, n_items * sizeof(int), s);
    if (e != cudaSuccess) return e;
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
