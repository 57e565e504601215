// Fifth link probe: does spreading each direction over several streams
// (copy engines) raise both-ways PCIe throughput for the connector geometry
// (64 x 1 MiB pieces per layer, strided 80 MiB apart on the host)?
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

int main() {
  CK(cudaSetDevice(0));
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  std::printf("asyncEngineCount=%d\n", pr.asyncEngineCount);
  // PIECE_MB: MiB per piece (a piece = that many consecutive layers of one
  // chunk, which are contiguous in a slot); the total moved stays 2.5 GiB.
  const int pm = std::getenv("PIECE_MB") ? std::atoi(std::getenv("PIECE_MB")) : 1;
  const int L = 40 / pm, N = 64;
  const size_t piece = size_t(pm) << 20, layer = N * piece, total = L * layer;
  char *dh, *dd, *hh, *hd;
  CK(cudaMalloc(&dh, total)); CK(cudaMalloc(&dd, total));
  CK(cudaHostAlloc((void**)&hh, total, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostAlloc((void**)&hd, total, cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(hh, 1, total); std::memset(hd, 2, total);
  auto hoff = [&](int l, int i) { return size_t(i) * L * piece + size_t(l) * piece; };
  const int MAXS = 4;
  cudaStream_t a[MAXS], b[MAXS];
  for (int i = 0; i < MAXS; ++i) { CK(cudaStreamCreateWithFlags(&a[i], cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&b[i], cudaStreamNonBlocking)); }
  cudaEvent_t t0, t1, j; CK(cudaEventCreate(&t0)); CK(cudaEventCreate(&t1)); CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
  cudaMemcpyAttributes attr{}; attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  size_t zero = 0, fail = 0;
  for (int ns : {1}) {
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(t0, a[0]));
      for (int s = 0; s < ns; ++s) { CK(cudaStreamWaitEvent(a[s], t0)); CK(cudaStreamWaitEvent(b[s], t0)); }
      for (int l = 0; l < L; ++l) {
        for (int s = 0; s < ns; ++s) {
          std::vector<void*> d1, s1, d2, s2; std::vector<size_t> sz;
          for (int i = s; i < N; i += ns) {
            d1.push_back(dh + l * layer + i * piece); s1.push_back(hh + hoff(l, i));
            d2.push_back(hd + hoff(l, i)); s2.push_back(dd + l * layer + i * piece); sz.push_back(piece);
          }
          CK(cudaMemcpyBatchAsync(d1.data(), s1.data(), sz.data(), d1.size(), &attr, &zero, 1, &fail, a[s]));
          CK(cudaMemcpyBatchAsync(d2.data(), s2.data(), sz.data(), d2.size(), &attr, &zero, 1, &fail, b[s]));
        }
      }
      for (int s = 0; s < ns; ++s) { CK(cudaEventRecord(j, a[s])); CK(cudaStreamWaitEvent(a[0], j)); CK(cudaEventRecord(j, b[s])); CK(cudaStreamWaitEvent(a[0], j)); }
      CK(cudaEventRecord(t1, a[0])); CK(cudaEventSynchronize(t1));
      float ms; CK(cudaEventElapsedTime(&ms, t0, t1));
      std::printf("piece=%d MiB streams/dir=%d both ways strided batches ms=%8.2f GBps=%6.1f\n", pm, ns, ms,
                  2.0 * total / ms / 1e6);
    }
  }
  return 0;
}
