// Does a pitched copy whose pitch x rows extent reaches past the end of its
// pinned host allocation (while every row it copies lies inside) succeed?
// csrc/ce_copy.cpp splits the last row off each run on the assumption that
// it may not. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probe_pitch_extent.cu -o build/ppe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <sys/mman.h>

int main() {
  const size_t slot = 40 << 10, w = 8 << 10, nslots = 48, rows = 8;
  char *h, *d;
  cudaHostAlloc((void**)&h, slot * nslots, cudaHostAllocPortable);
  cudaMalloc(&d, rows * w);
  std::memset(h, 7, slot * nslots);
  cudaStream_t s; cudaStreamCreate(&s);
  const char* src = h + (nslots - rows) * slot;  // last row = first bytes of the last slot
  cudaError_t e1 = cudaMemcpy2DAsync(d, w, src, slot, w, rows, cudaMemcpyHostToDevice, s);
  cudaError_t e1s = cudaStreamSynchronize(s);
  cudaGetLastError();
  cudaError_t e2 = cudaMemcpy2DAsync((void*)src, slot, d, w, w, rows, cudaMemcpyDeviceToHost, s);
  cudaError_t e2s = cudaStreamSynchronize(s);
  cudaGetLastError();
  cudaError_t e3 = cudaMemcpy2DAsync(d, w, h, slot, w, rows, cudaMemcpyHostToDevice, s);  // inside
  cudaError_t e3s = cudaStreamSynchronize(s);
  // the same past-end extent on registered memory (mmap + cudaHostRegister, as
  // the tier slab may be): the bytes past the registration are unregistered
  char* m = (char*)mmap(nullptr, slot * nslots + (2 << 20), PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  cudaError_t er = cudaHostRegister(m, slot * nslots, cudaHostRegisterMapped | cudaHostRegisterPortable);
  const char* msrc = m + (nslots - rows) * slot;
  cudaError_t e4 = cudaMemcpy2DAsync(d, w, msrc, slot, w, rows, cudaMemcpyHostToDevice, s);
  cudaError_t e4s = cudaStreamSynchronize(s);
  cudaGetLastError();
  cudaError_t e5 = cudaMemcpy2DAsync((void*)msrc, slot, d, w, w, rows, cudaMemcpyDeviceToHost, s);
  cudaError_t e5s = cudaStreamSynchronize(s);
  cudaGetLastError();
  std::printf("registered: %s\n", cudaGetErrorString(er));
  std::printf("registered h2d past-end extent: %s / %s\n", cudaGetErrorString(e4), cudaGetErrorString(e4s));
  std::printf("registered d2h past-end extent: %s / %s\n", cudaGetErrorString(e5), cudaGetErrorString(e5s));
  std::printf("h2d past-end extent: %s / %s\n", cudaGetErrorString(e1), cudaGetErrorString(e1s));
  std::printf("d2h past-end extent: %s / %s\n", cudaGetErrorString(e2), cudaGetErrorString(e2s));
  std::printf("h2d inside extent:   %s / %s\n", cudaGetErrorString(e3), cudaGetErrorString(e3s));
  return 0;
}
