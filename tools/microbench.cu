// Link-roofline probe for the KV data-movement path on one B200.
//   HBM:   16-byte vectorised device copy kernel vs cudaMemcpyAsync D2D
//   PCIe:  pinned cudaMemcpyAsync H2D / D2H / both directions at once
//   UVA:   kernel loads from / stores to mapped pinned host memory (the
//          zero-copy path the fused gather/scatter kernels would use)
// Prints one line per measurement: name, bytes, ms, GB/s.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

template <int UNROLL>
__global__ void copy16(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t stride = size_t(gridDim.x) * blockDim.x * UNROLL;
  for (size_t base = size_t(blockIdx.x) * blockDim.x * UNROLL + threadIdx.x; base < n16; base += stride) {
    int4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      size_t i = base + size_t(u) * blockDim.x;
      if (i < n16) v[u] = src[i];
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      size_t i = base + size_t(u) * blockDim.x;
      if (i < n16) dst[i] = v[u];
    }
  }
}

static float time_it(cudaStream_t s, int reps, auto&& fn) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  fn(); CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(a, s));
  for (int i = 0; i < reps; ++i) fn();
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms = 0; CK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a); cudaEventDestroy(b);
  return ms / reps;
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  std::printf("device %s sms=%d l2=%d MiB\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20);
  const size_t bytes = size_t(1) << 30;
  void *d0, *d1, *h0, *h1;
  CK(cudaMalloc(&d0, bytes)); CK(cudaMalloc(&d1, bytes));
  CK(cudaHostAlloc(&h0, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostAlloc(&h1, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaMemset(d0, 1, bytes)); CK(cudaMemset(d1, 2, bytes));
  std::vector<char> tmp(bytes, 3);
  std::memcpy(h0, tmp.data(), bytes); std::memcpy(h1, tmp.data(), bytes);
  void *hd0, *hd1;
  CK(cudaHostGetDevicePointer(&hd0, h0, 0)); CK(cudaHostGetDevicePointer(&hd1, h1, 0));
  cudaStream_t s, s2; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  const size_t n16 = bytes / 16;
  auto rep = [&](const char* name, double moved, float ms) {
    std::printf("%-40s bytes=%.0f ms=%.3f GBps=%.1f\n", name, moved, ms, moved / ms / 1e6);
  };

  // HBM: counted read+write like MEASURED_PEAKS.json.
  float ms = time_it(s, 10, [&] { CK(cudaMemcpyAsync(d1, d0, bytes, cudaMemcpyDeviceToDevice, s)); });
  rep("hbm memcpy d2d (r+w)", 2.0 * bytes, ms);
  for (int blocks : {148, 296, 592, 1184, 2368}) {
    for (int threads : {256, 512}) {
      ms = time_it(s, 10, [&] { copy16<4><<<blocks, threads, 0, s>>>((const int4*)d0, (int4*)d1, n16); });
      char nm[96]; std::snprintf(nm, sizeof nm, "hbm copy16<4> g=%d t=%d (r+w)", blocks, threads);
      rep(nm, 2.0 * bytes, ms);
      ms = time_it(s, 10, [&] { copy16<8><<<blocks, threads, 0, s>>>((const int4*)d0, (int4*)d1, n16); });
      std::snprintf(nm, sizeof nm, "hbm copy16<8> g=%d t=%d (r+w)", blocks, threads);
      rep(nm, 2.0 * bytes, ms);
    }
  }

  // PCIe copy engines.
  ms = time_it(s, 5, [&] { CK(cudaMemcpyAsync(d0, h0, bytes, cudaMemcpyHostToDevice, s)); });
  rep("pcie memcpy h2d", bytes, ms);
  ms = time_it(s, 5, [&] { CK(cudaMemcpyAsync(h1, d1, bytes, cudaMemcpyDeviceToHost, s)); });
  rep("pcie memcpy d2h", bytes, ms);
  {
    cudaEvent_t a, b, j; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&j));
    CK(cudaEventRecord(a, s)); CK(cudaStreamWaitEvent(s2, a));
    for (int i = 0; i < 5; ++i) {
      CK(cudaMemcpyAsync(d0, h0, bytes, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(h1, d1, bytes, cudaMemcpyDeviceToHost, s2));
    }
    CK(cudaEventRecord(j, s2)); CK(cudaStreamWaitEvent(s, j)); CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
    rep("pcie memcpy bidir (h2d+d2h)", 10.0 * bytes, ms);
  }
  // Chunk-layer sized copies (1 MiB) as the layerwise path would issue.
  ms = time_it(s, 3, [&] {
    for (size_t off = 0; off < bytes; off += (1 << 20))
      CK(cudaMemcpyAsync((char*)d0 + off, (char*)h0 + off, 1 << 20, cudaMemcpyHostToDevice, s));
  });
  rep("pcie memcpy h2d 1MiB pieces", bytes, ms);

  // Zero-copy kernels over mapped pinned memory.
  for (int blocks : {148, 296, 592, 1184}) {
    for (int threads : {256, 512}) {
      char nm[96];
      ms = time_it(s, 3, [&] { copy16<4><<<blocks, threads, 0, s>>>((const int4*)hd0, (int4*)d0, n16); });
      std::snprintf(nm, sizeof nm, "uva read host->dev g=%d t=%d", blocks, threads);
      rep(nm, bytes, ms);
      ms = time_it(s, 3, [&] { copy16<4><<<blocks, threads, 0, s>>>((const int4*)d1, (int4*)hd1, n16); });
      std::snprintf(nm, sizeof nm, "uva write dev->host g=%d t=%d", blocks, threads);
      rep(nm, bytes, ms);
    }
  }
  {
    cudaEvent_t a, b, j; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&j));
    for (int blocks : {148, 296, 592}) {
      CK(cudaEventRecord(a, s)); CK(cudaStreamWaitEvent(s2, a));
      for (int i = 0; i < 3; ++i) {
        copy16<4><<<blocks, 512, 0, s>>>((const int4*)hd0, (int4*)d0, n16);
        copy16<4><<<blocks, 512, 0, s2>>>((const int4*)d1, (int4*)hd1, n16);
      }
      CK(cudaEventRecord(j, s2)); CK(cudaStreamWaitEvent(s, j)); CK(cudaEventRecord(b, s));
      CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
      char nm[96]; std::snprintf(nm, sizeof nm, "uva bidir g=%d each", blocks);
      rep(nm, 6.0 * bytes, ms);
    }
  }
  std::printf("done\n");
  return 0;
}
