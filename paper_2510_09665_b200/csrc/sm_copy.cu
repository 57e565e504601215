// SM-driven copy between any two device-visible addresses (HBM, mapped pinned
// host memory, a peer GPU's memory). Small per-step uploads issued by the
// engine (its prompt tokens) must not queue on the copy engines behind
// ~100 ms of layerwise KV transfers; a kernel reading pinned
// memory over PCIe is scheduled on the SMs instead and lands in microseconds.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace tkv {
namespace {

// 16-byte body plus the (< 16 byte) tail in the same launch.
__global__ void __launch_bounds__(256)
sm_copy16_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t n16, uint32_t tail) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
         i += uint64_t(gridDim.x) * blockDim.x)
        dst[i] = src[i];
    if (blockIdx.x == 0 && threadIdx.x < tail)
        reinterpret_cast<uint8_t*>(dst + n16)[threadIdx.x] = reinterpret_cast<const uint8_t*>(src + n16)[threadIdx.x];
}

__global__ void __launch_bounds__(256)
sm_copy1_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

int grid_for(uint64_t items) {
    const uint64_t g = (items + 255) / 256;
    return int(g < 148 * 4 ? (g ? g : 1) : 148 * 4);
}

}  // namespace

cudaError_t launch_sm_copy(const void* src, void* dst, uint64_t bytes, cudaStream_t s) {
    if (bytes == 0) return cudaSuccess;
    const auto* s8 = static_cast<const uint8_t*>(src);
    auto* d8 = static_cast<uint8_t*>(dst);
    uint64_t body = 0;
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        note_launch();
        sm_copy16_kernel<<<grid_for(bytes / 16), 256, 0, s>>>(reinterpret_cast<const uint4*>(s8),
                                                               reinterpret_cast<uint4*>(d8), bytes / 16,
                                                               uint32_t(bytes & 15));
        return cudaGetLastError();
    }
    if (bytes > body) {
        note_launch();
        sm_copy1_kernel<<<grid_for(bytes - body), 256, 0, s>>>(s8 + body, d8 + body, bytes - body);
    }
    return cudaGetLastError();
}

}  // namespace tkv
