#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cstdlib>
double now() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  const size_t n = 512 * 1024;
  std::vector<char> src(n, 1);
  std::vector<char> dst1(n);
  void* pinned = nullptr; cudaHostAlloc(&pinned, n, cudaHostAllocMapped | cudaHostAllocPortable);
  void* wc = nullptr; cudaHostAlloc(&wc, n, cudaHostAllocMapped | cudaHostAllocWriteCombined);
  char* m = (char*)aligned_alloc(4096, n); cudaHostRegister(m, n, cudaHostRegisterMapped);
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now(); memcpy(dst1.data(), src.data(), n); double t1 = now();
    memcpy(pinned, src.data(), n); double t2 = now();
    memcpy(m, src.data(), n); double t3 = now();
    memcpy(wc, src.data(), n); double t4 = now();
    printf("pageable %.1f us | cudaHostAlloc %.1f us | registered %.1f us | write-combined %.1f us\n", t1-t0, t2-t1, t3-t2, t4-t3);
  }
  return 0;
}
