// Host-tier link probe for the connector geometry: per layer 64 pieces of
// PIECE_KB KiB (one chunk-layer slice each), strided one slot apart on the
// host (slot layout [L][T][bpt]), packed in the HBM ring; 40 layers. Each
// layer goes to the copy engine as
//   piece : one cudaMemcpyAsync per piece
//   2d    : one cudaMemcpy2DAsync per layer (width = piece, height = 64,
//           host pitch = slot bytes) -- what csrc/ce_copy.cpp issues for a
//           run of consecutive slots
//   one   : a single large contiguous copy of the same bytes (upper bound)
//   split : as 2d, but each layer's D2H in two pitched copies (56 + 8 rows:
//           a store batch whose slots are two runs)
// in H2D only, D2H only, and both directions at once.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench_pitched.cu -o /tmp/mbp
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

int main() {
  CK(cudaSetDevice(0));
  const int pk = std::getenv("PIECE_KB") ? std::atoi(std::getenv("PIECE_KB")) : 1024;
  const int L = std::getenv("LAYERS") ? std::atoi(std::getenv("LAYERS")) : 40, N = 64;
  const size_t piece = size_t(pk) << 10, layer = size_t(N) * piece, total = size_t(L) * layer;
  const size_t slot = size_t(L) * piece;  // one chunk's [L][T][bpt] payload
  char *dh, *dd, *hh, *hd;
  CK(cudaMalloc(&dh, total)); CK(cudaMalloc(&dd, total));
  CK(cudaHostAlloc((void**)&hh, total, cudaHostAllocPortable));
  CK(cudaHostAlloc((void**)&hd, total, cudaHostAllocPortable));
  std::memset(hh, 1, total); std::memset(hd, 2, total);
  cudaStream_t a, b;
  CK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
  cudaEvent_t t0, t1, j; CK(cudaEventCreate(&t0)); CK(cudaEventCreate(&t1)); CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
  auto h2d = [&](int mode, int l) {
    if (mode == 0) for (int i = 0; i < N; ++i)
      CK(cudaMemcpyAsync(dh + l * layer + i * piece, hh + i * slot + l * piece, piece, cudaMemcpyHostToDevice, a));
    else if (mode == 1 || mode == 3)
      CK(cudaMemcpy2DAsync(dh + l * layer, piece, hh + l * piece, slot, piece, N, cudaMemcpyHostToDevice, a));
    else CK(cudaMemcpyAsync(dh + l * layer, hh + l * layer, layer, cudaMemcpyHostToDevice, a));
  };
  auto d2h = [&](int mode, int l) {
    if (mode == 0) for (int i = 0; i < N; ++i)
      CK(cudaMemcpyAsync(hd + i * slot + l * piece, dd + l * layer + i * piece, piece, cudaMemcpyDeviceToHost, b));
    else if (mode == 1)
      CK(cudaMemcpy2DAsync(hd + l * piece, slot, dd + l * layer, piece, piece, N, cudaMemcpyDeviceToHost, b));
    else if (mode == 3) {
      CK(cudaMemcpy2DAsync(hd + l * piece, slot, dd + l * layer, piece, piece, N - 8, cudaMemcpyDeviceToHost, b));
      CK(cudaMemcpy2DAsync(hd + (N - 8) * slot + l * piece, slot, dd + l * layer + (N - 8) * piece, piece, piece, 8,
                           cudaMemcpyDeviceToHost, b));
    }
    else CK(cudaMemcpyAsync(hd + l * layer, dd + l * layer, layer, cudaMemcpyDeviceToHost, b));
  };
  const char* names[] = {"piece", "2d", "one", "split"};
  const char* dirs[] = {"h2d", "d2h", "both"};
  for (int mode = 0; mode < 4; ++mode)
    for (int dir = 0; dir < 3; ++dir)
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(t0, a)); CK(cudaStreamWaitEvent(b, t0));
        for (int l = 0; l < L; ++l) {
          if (dir != 1) h2d(mode, l);
          if (dir != 0) d2h(mode, l);
        }
        CK(cudaEventRecord(j, b)); CK(cudaStreamWaitEvent(a, j));
        CK(cudaEventRecord(t1, a)); CK(cudaEventSynchronize(t1));
        float ms; CK(cudaEventElapsedTime(&ms, t0, t1));
        const double bytes = (dir == 2 ? 2.0 : 1.0) * total;
        std::printf("piece=%dKiB mode=%-5s dir=%-4s ms=%8.2f GBps=%6.1f\n", pk, names[mode], dirs[dir], ms, bytes / ms / 1e6);
      }
  return 0;
}
