// q8-scale codec on the device, bit-exact with
// Q8ScaleCodec (src/codec.cpp:27-91):
//   payload = signed 16-bit little-endian lanes (+ a raw odd tail byte)
//   scale   = float(max|lane| / 127.0)            (q8_scale_of, codec.cpp:86-94)
//   encode  = round(double(lane) / double(scale)) clamped to [-127, 127], int8
//   decode  = round(double(q) * double(scale)) clamped to [-32768, 32767]
//   blob    = u32le original_len | f32le scale | int8 lanes | odd tail byte
// round() is round-half-away-from-zero in both C and CUDA, and double
// division / multiplication are IEEE correctly rounded on both sides, so the
// bytes match. One launch covers a batch of chunk payloads; HBM-bound
// (encode reads the payload twice — absmax, then quantise — and writes half).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace tkv {
namespace {

constexpr int kThreads = 256;
constexpr uint64_t kSeg = 64 * 1024;  // payload bytes per CTA work item

__device__ __forceinline__ int32_t lane16(uint32_t w, int half) {
    return int32_t(int16_t(uint16_t(w >> (16 * half))));
}

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
        if ((reinterpret_cast<uint64_t>(it.src) & 3) == 0) {
            for (uint64_t b = b0 + 4 * threadIdx.x; b + 4 <= b1; b += 4 * kThreads) {
                const uint32_t w = __ldcs(reinterpret_cast<const unsigned int*>(it.src + b));
                m = max(m, max(abs(lane16(w, 0)), abs(lane16(w, 1))));
            }
            // a 2-byte lane left over when (b1 - b0) % 4 == 2
            const uint64_t tail = b0 + ((b1 - b0) & ~uint64_t(3));
            if (threadIdx.x == 0 && tail + 2 <= b1)
                m = max(m, abs(int32_t(int16_t(uint16_t(it.src[tail] | (it.src[tail + 1] << 8))))));
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

__device__ __forceinline__ uint32_t quant(int32_t lane, float scale) {
    double q = scale > 0.f ? round(double(lane) / double(scale)) : 0.0;
    q = fmin(127.0, fmax(-127.0, q));
    return uint32_t(uint8_t(int8_t(q)));
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
        for (uint64_t b = b0 + 2 * threadIdx.x; b + 2 <= b1; b += 2 * kThreads) {
            const int32_t lane = int32_t(int16_t(uint16_t(it.src[b] | (it.src[b + 1] << 8))));
            out[b / 2] = uint8_t(quant(lane, scale));
        }
    }
}

__global__ void __launch_bounds__(kThreads)
q8_decode_kernel(const CodecItem* __restrict__ items, const uint32_t* __restrict__ seg_base,
                 uint32_t n_items, uint32_t total_segs) {
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
        for (uint64_t b = b0 + 2 * threadIdx.x; b + 2 <= b1; b += 2 * kThreads) {
            const int8_t q = int8_t(it.src[8 + b / 2]);
            double v = round(double(q) * double(scale));
            v = fmin(32767.0, fmax(-32768.0, v));
            const uint16_t lane = uint16_t(int16_t(v));
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
