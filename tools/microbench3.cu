// Third link probe: does copy-engine concurrency between directions survive
// the connector's submission pattern?
//   a) 80 H2D batches (64 x 1 MiB) enqueued first, then 80 D2H batches
//   b) the same batches interleaved in submission order
//   c) like a) but one cudaMemcpyAsync per piece
//   d) like b) with per-piece cudaMemcpyAsync
//   e) one 5 GiB H2D + one 5 GiB D2H (upper bound)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

int main() {
  CK(cudaSetDevice(0));
  const int L = 80, N = 64;
  const size_t piece = 1 << 20, layer = N * piece, total = L * layer;  // 5 GiB
  char *dh, *dd, *hh, *hd;
  CK(cudaMalloc(&dh, total)); CK(cudaMalloc(&dd, total));
  CK(cudaHostAlloc((void**)&hh, total, cudaHostAllocMapped)); CK(cudaHostAlloc((void**)&hd, total, cudaHostAllocMapped));
  std::memset(hh, 1, total); std::memset(hd, 2, total);
  cudaStream_t a, b; CK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
  cudaEvent_t t0, t1, j; CK(cudaEventCreate(&t0)); CK(cudaEventCreate(&t1)); CK(cudaEventCreate(&j));
  cudaMemcpyAttributes attr{}; attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  size_t zero = 0, fail = 0;
  std::vector<void*> hd_dst(N), hd_src(N), dh_dst(N), dh_src(N); std::vector<size_t> sz(N, piece);
  auto h2d = [&](int l, bool batch) {
    for (int i = 0; i < N; ++i) { hd_dst[i] = dh + l * layer + i * piece; hd_src[i] = hh + l * layer + i * piece; }
    if (batch) CK(cudaMemcpyBatchAsync(hd_dst.data(), hd_src.data(), sz.data(), N, &attr, &zero, 1, &fail, a));
    else for (int i = 0; i < N; ++i) CK(cudaMemcpyAsync(hd_dst[i], hd_src[i], piece, cudaMemcpyHostToDevice, a));
  };
  auto d2h = [&](int l, bool batch) {
    for (int i = 0; i < N; ++i) { dh_dst[i] = hd + l * layer + i * piece; dh_src[i] = dd + l * layer + i * piece; }
    if (batch) CK(cudaMemcpyBatchAsync(dh_dst.data(), dh_src.data(), sz.data(), N, &attr, &zero, 1, &fail, b));
    else for (int i = 0; i < N; ++i) CK(cudaMemcpyAsync(dh_dst[i], dh_src[i], piece, cudaMemcpyDeviceToHost, b));
  };
  auto run = [&](const char* name, auto&& body) {
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(t0, a)); CK(cudaStreamWaitEvent(b, t0));
    body();
    CK(cudaEventRecord(j, b)); CK(cudaStreamWaitEvent(a, j)); CK(cudaEventRecord(t1, a));
    CK(cudaEventSynchronize(t1)); float ms; CK(cudaEventElapsedTime(&ms, t0, t1));
    std::printf("%-44s ms=%8.2f GBps(sum)=%6.1f\n", name, ms, 2.0 * total / ms / 1e6);
  };
  for (int rep = 0; rep < 2; ++rep) {
    run("a) batch: all H2D first, then all D2H", [&] { for (int l = 0; l < L; ++l) h2d(l, true); for (int l = 0; l < L; ++l) d2h(l, true); });
    run("b) batch: interleaved", [&] { for (int l = 0; l < L; ++l) { h2d(l, true); d2h(l, true); } });
    run("c) per-piece: all H2D first, then all D2H", [&] { for (int l = 0; l < L; ++l) h2d(l, false); for (int l = 0; l < L; ++l) d2h(l, false); });
    run("d) per-piece: interleaved", [&] { for (int l = 0; l < L; ++l) { h2d(l, false); d2h(l, false); } });
    run("e) one 5 GiB copy each way", [&] { CK(cudaMemcpyAsync(dh, hh, total, cudaMemcpyHostToDevice, a)); CK(cudaMemcpyAsync(hd, dd, total, cudaMemcpyDeviceToHost, b)); });
    run("f) batch: D2H lags H2D by 1 (event chain)", [&] {
      std::vector<cudaEvent_t> ev(L);
      for (int l = 0; l < L; ++l) { CK(cudaEventCreateWithFlags(&ev[l], cudaEventDisableTiming)); }
      for (int l = 0; l < L; ++l) { h2d(l, true); CK(cudaEventRecord(ev[l], a)); }
      for (int l = 0; l < L; ++l) { CK(cudaStreamWaitEvent(b, ev[l])); d2h(l, true); }
    });
  }
  std::printf("done\n");
  return 0;
}
