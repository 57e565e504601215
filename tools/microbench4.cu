// Fourth link probe: does the HOST allocation change PCIe throughput?
//   A) cudaHostAlloc(Mapped|Portable)           (what TieredStore uses)
//   B) 2 MiB-aligned mmap + MADV_HUGEPAGE + cudaHostRegister(Mapped|Portable)
//   C) cudaHostAlloc(WriteCombined) for the H2D source
// For each: H2D alone, D2H alone, both directions at once, with 64 x 1 MiB
// cudaMemcpyBatchAsync per "layer" (the connector's pattern) and one big copy.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

static char* huge_host(size_t bytes) {
  const size_t align = 2u << 20;
  void* p = mmap(nullptr, bytes + align, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) { std::perror("mmap"); std::exit(1); }
  char* a = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + align - 1) & ~(align - 1));
  if (madvise(a, bytes, MADV_HUGEPAGE) != 0) std::perror("madvise");
  std::memset(a, 3, bytes);
  CK(cudaHostRegister(a, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
  return a;
}

int main() {
  CK(cudaSetDevice(0));
  const int L = 40, N = 64;
  const size_t piece = 1 << 20, layer = N * piece, total = L * layer;  // 2.5 GiB per direction
  // STRIDED=1: the connector's geometry — piece i of layer l at slot i
  // (slot = L MiB), offset l MiB (chunk payload [L][T][bpt]).
  const bool strided = std::getenv("STRIDED") != nullptr;
  auto hoff = [&](int l, int i) { return strided ? size_t(i) * L * piece + size_t(l) * piece : l * layer + i * piece; };
  char *dh, *dd;
  CK(cudaMalloc(&dh, total)); CK(cudaMalloc(&dd, total));
  cudaStream_t a, b; CK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
  cudaEvent_t t0, t1, j; CK(cudaEventCreate(&t0)); CK(cudaEventCreate(&t1)); CK(cudaEventCreate(&j));
  cudaMemcpyAttributes attr{}; attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  size_t zero = 0, fail = 0;
  std::vector<void*> d1(N), s1(N), d2(N), s2(N); std::vector<size_t> sz(N, piece);
  struct Alloc { const char* name; char* hh; char* hd; };
  std::vector<Alloc> allocs;
  {
    char *x, *y; CK(cudaHostAlloc((void**)&x, total, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaHostAlloc((void**)&y, total, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(x, 1, total); std::memset(y, 2, total);
    allocs.push_back({"A cudaHostAlloc", x, y});
  }
  allocs.push_back({"B mmap+THP+register", huge_host(total), huge_host(total)});
  {
    char* x; CK(cudaHostAlloc((void**)&x, total, cudaHostAllocWriteCombined | cudaHostAllocMapped));
    std::memset(x, 1, total);
    allocs.push_back({"C WC h2d src, A d2h dst", x, allocs[0].hd});
  }
  for (auto& al : allocs) {
    auto h2d = [&](int l) {
      for (int i = 0; i < N; ++i) { d1[i] = dh + l * layer + i * piece; s1[i] = al.hh + hoff(l, i); }
      CK(cudaMemcpyBatchAsync(d1.data(), s1.data(), sz.data(), N, &attr, &zero, 1, &fail, a));
    };
    auto d2h = [&](int l) {
      for (int i = 0; i < N; ++i) { d2[i] = al.hd + hoff(l, i); s2[i] = dd + l * layer + i * piece; }
      CK(cudaMemcpyBatchAsync(d2.data(), s2.data(), sz.data(), N, &attr, &zero, 1, &fail, b));
    };
    auto run = [&](const char* what, double bytes, auto&& body) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(t0, a)); CK(cudaStreamWaitEvent(b, t0));
      body();
      CK(cudaEventRecord(j, b)); CK(cudaStreamWaitEvent(a, j)); CK(cudaEventRecord(t1, a));
      CK(cudaEventSynchronize(t1)); float ms; CK(cudaEventElapsedTime(&ms, t0, t1));
      std::printf("%-26s %-28s ms=%8.2f GBps=%6.1f\n", al.name, what, ms, bytes / ms / 1e6);
    };
    for (int rep = 0; rep < 2; ++rep) {
      run("h2d batches", total, [&] { for (int l = 0; l < L; ++l) h2d(l); });
      run("d2h batches", total, [&] { for (int l = 0; l < L; ++l) d2h(l); });
      run("both batches interleaved", 2.0 * total, [&] { for (int l = 0; l < L; ++l) { h2d(l); d2h(l); } });
      run("both one copy each", 2.0 * total, [&] {
        CK(cudaMemcpyAsync(dh, al.hh, total, cudaMemcpyHostToDevice, a));
        CK(cudaMemcpyAsync(al.hd, dd, total, cudaMemcpyDeviceToHost, b)); });
    }
  }
  std::printf("done\n");
  return 0;
}
