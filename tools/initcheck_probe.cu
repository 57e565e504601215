#include <cuda_runtime.h>
#include <cstdio>
__global__ void rd(const int4* p, int n, int* out) { int s = 0; for (int i = threadIdx.x; i < n; i += blockDim.x) s += p[i].x; atomicAdd(out, s); }
int main() {
  const size_t n = 1 << 20; char *h, *d1, *d2; int* o;
  cudaHostAlloc(&h, n, cudaHostAllocMapped); for (size_t i = 0; i < n; ++i) h[i] = char(i);
  cudaMalloc(&d1, n); cudaMalloc(&d2, n); cudaMalloc(&o, 4); cudaMemset(o, 0, 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaMemcpyAsync(d1, h, n, cudaMemcpyHostToDevice, s);
  void* dst[1] = {d2}; void* src[1] = {h}; size_t sz[1] = {n};
  cudaMemcpyAttributes attr{}; attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream; size_t zero = 0, fail = 0;
  cudaMemcpyBatchAsync(dst, src, sz, 1, &attr, &zero, 1, &fail, s);
  rd<<<1, 256, 0, s>>>((const int4*)d1, n / 16, o);  // plain memcpy'd
  cudaStreamSynchronize(s); printf("after plain memcpy read\n"); fflush(stdout);
  rd<<<1, 256, 0, s>>>((const int4*)d2, n / 16, o);  // batch memcpy'd
  cudaStreamSynchronize(s); printf("done\n");
}
