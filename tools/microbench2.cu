// Second link probe: how the host tier should be driven.
//   CE pieces:   per-piece cudaMemcpyAsync vs one cudaMemcpyBatchAsync, for the
//                chunk-layer slice sizes of the configs (1 MiB at 8B/70B TP=1,
//                128 KiB at 70B TP=8), one direction and both at once.
//   hybrid:      copy engine one way + zero-copy kernel the other way.
//   small grids: zero-copy bandwidth with few CTAs (leaves SMs to compute).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <functional>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

__global__ void copy16(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  constexpr int U = 4;
  size_t stride = size_t(gridDim.x) * blockDim.x * U;
  for (size_t base = size_t(blockIdx.x) * blockDim.x * U + threadIdx.x; base < n16; base += stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t i = base + size_t(u) * blockDim.x; if (i < n16) v[u] = src[i]; }
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t i = base + size_t(u) * blockDim.x; if (i < n16) dst[i] = v[u]; }
  }
}

struct Timer {
  cudaEvent_t a, b;
  Timer() { CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); }
  void start(cudaStream_t s) { CK(cudaEventRecord(a, s)); }
  float stop(cudaStream_t s) { CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b)); return ms; }
};

int main() {
  CK(cudaSetDevice(0));
  const size_t bytes = size_t(1) << 30;
  char *d0, *d1, *h0, *h1;
  CK(cudaMalloc(&d0, 2 * bytes)); CK(cudaMalloc(&d1, 2 * bytes));
  CK(cudaHostAlloc((void**)&h0, 2 * bytes, cudaHostAllocMapped)); CK(cudaHostAlloc((void**)&h1, 2 * bytes, cudaHostAllocMapped));
  std::memset(h0, 1, 2 * bytes); std::memset(h1, 2, 2 * bytes);
  CK(cudaMemset(d0, 0, 2 * bytes)); CK(cudaMemset(d1, 0, 2 * bytes));
  char *hd0, *hd1; CK(cudaHostGetDevicePointer((void**)&hd0, h0, 0)); CK(cudaHostGetDevicePointer((void**)&hd1, h1, 0));
  cudaStream_t s, s2; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t fork, join; CK(cudaEventCreate(&fork)); CK(cudaEventCreate(&join));
  Timer t;
  auto rep = [](const char* nm, double b, float ms) { std::printf("%-52s ms=%8.3f GBps=%6.1f\n", nm, ms, b / ms / 1e6); };

  cudaMemcpyAttributes attr{}; attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  for (size_t piece : {size_t(128) << 10, size_t(256) << 10, size_t(1) << 20, size_t(4) << 20}) {
    size_t n = bytes / piece;
    // scattered: piece i lands at stride 2*piece (slot-like placement)
    std::vector<void*> dh(n), sh(n), dd(n), sd(n); std::vector<size_t> sz(n, piece);
    for (size_t i = 0; i < n; ++i) {
      dh[i] = d0 + 2 * i * piece; sh[i] = h0 + 2 * i * piece;     // h2d
      dd[i] = h1 + 2 * i * piece; sd[i] = d1 + 2 * i * piece;     // d2h
    }
    auto h2d_loop = [&](cudaStream_t st) { for (size_t i = 0; i < n; ++i) CK(cudaMemcpyAsync(dh[i], sh[i], piece, cudaMemcpyHostToDevice, st)); };
    auto d2h_loop = [&](cudaStream_t st) { for (size_t i = 0; i < n; ++i) CK(cudaMemcpyAsync(dd[i], sd[i], piece, cudaMemcpyDeviceToHost, st)); };
    size_t fail = 0, zero = 0;
    auto h2d_batch = [&](cudaStream_t st) { CK(cudaMemcpyBatchAsync(dh.data(), sh.data(), sz.data(), n, &attr, &zero, 1, &fail, st)); };
    auto d2h_batch = [&](cudaStream_t st) { CK(cudaMemcpyBatchAsync(dd.data(), sd.data(), sz.data(), n, &attr, &zero, 1, &fail, st)); };
    char nm[128];
    for (int mode = 0; mode < 2; ++mode) {
      std::function<void(cudaStream_t)> h2d = h2d_loop, d2h = d2h_loop; if (mode) { h2d = h2d_batch; d2h = d2h_batch; }
      const char* mn = mode ? "batch" : "loop";
      h2d(s); CK(cudaStreamSynchronize(s));
      t.start(s); for (int r = 0; r < 3; ++r) h2d(s); float ms = t.stop(s) / 3;
      std::snprintf(nm, sizeof nm, "ce h2d %s piece=%zuK", mn, piece >> 10); rep(nm, bytes, ms);
      t.start(s); for (int r = 0; r < 3; ++r) d2h(s); ms = t.stop(s) / 3;
      std::snprintf(nm, sizeof nm, "ce d2h %s piece=%zuK", mn, piece >> 10); rep(nm, bytes, ms);
      t.start(s); CK(cudaStreamWaitEvent(s2, t.a));
      for (int r = 0; r < 3; ++r) { h2d(s); d2h(s2); }
      CK(cudaEventRecord(join, s2)); CK(cudaStreamWaitEvent(s, join)); ms = t.stop(s) / 3;
      std::snprintf(nm, sizeof nm, "ce bidir %s piece=%zuK (sum)", mn, piece >> 10); rep(nm, 2.0 * bytes, ms);
    }
  }
  // Hybrid: CE h2d + zero-copy kernel d2h, and zero-copy read + CE d2h.
  for (int g : {32, 74, 148}) {
    char nm[128]; float ms;
    t.start(s); CK(cudaStreamWaitEvent(s2, t.a));
    for (int r = 0; r < 3; ++r) { CK(cudaMemcpyAsync(d0, h0, bytes, cudaMemcpyHostToDevice, s)); copy16<<<g, 512, 0, s2>>>((const int4*)d1, (int4*)hd1, bytes / 16); }
    CK(cudaEventRecord(join, s2)); CK(cudaStreamWaitEvent(s, join)); ms = t.stop(s) / 3;
    std::snprintf(nm, sizeof nm, "hybrid ce-h2d + uva-write g=%d (sum)", g); rep(nm, 2.0 * bytes, ms);
    t.start(s); CK(cudaStreamWaitEvent(s2, t.a));
    for (int r = 0; r < 3; ++r) { copy16<<<g, 512, 0, s>>>((const int4*)hd0, (int4*)d0, bytes / 16); CK(cudaMemcpyAsync(h1, d1, bytes, cudaMemcpyDeviceToHost, s2)); }
    CK(cudaEventRecord(join, s2)); CK(cudaStreamWaitEvent(s, join)); ms = t.stop(s) / 3;
    std::snprintf(nm, sizeof nm, "hybrid uva-read + ce-d2h g=%d (sum)", g); rep(nm, 2.0 * bytes, ms);
  }
  for (int g : {8, 16, 32, 64}) {
    char nm[128];
    t.start(s); for (int r = 0; r < 3; ++r) copy16<<<g, 512, 0, s>>>((const int4*)hd0, (int4*)d0, bytes / 16); float ms = t.stop(s) / 3;
    std::snprintf(nm, sizeof nm, "uva read g=%d", g); rep(nm, bytes, ms);
    t.start(s); for (int r = 0; r < 3; ++r) copy16<<<g, 512, 0, s>>>((const int4*)d1, (int4*)hd1, bytes / 16); ms = t.stop(s) / 3;
    std::snprintf(nm, sizeof nm, "uva write g=%d", g); rep(nm, bytes, ms);
  }
  std::printf("done\n");
  return 0;
}
