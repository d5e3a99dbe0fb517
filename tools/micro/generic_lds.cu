// Latency of a dependent chain of shared-memory loads: ld.shared (LDS) vs generic ld (LD.E
// on a shared address).  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/glds generic_lds.cu
#include <cstdio>
#include <cstdint>

__global__ void chase(const int* __restrict__ init, int iters, int use_generic, long long* out,
                      int* sink, int** slot) {
  __shared__ int buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = init[i];
  __syncthreads();
  if (threadIdx.x == 0) *(int* volatile*)slot = buf;  // opaque generic pointer
  __syncthreads();
  int* g = *(int* volatile*)slot;
  int x = 0;
  long long t0 = clock64();
  if (use_generic) {
    for (int i = 0; i < iters; ++i) x = g[x];
  } else {
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(buf);
    for (int i = 0; i < iters; ++i)
      asm volatile("ld.shared.s32 %0, [%1];" : "=r"(x) : "r"(base + 4u * x));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[use_generic] = t1 - t0;
    sink[0] = x;
  }
}

int main() {
  int h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = (i * 37 + 11) & 1023;
  int *d, *sink;
  long long* o;
  int** slot;
  cudaMalloc(&slot, 8);
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&sink, 4);
  cudaMalloc(&o, 16);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    chase<<<1, 32>>>(d, 10000, 0, o, sink, slot);
    chase<<<1, 32>>>(d, 10000, 1, o, sink, slot);
    long long r[2];
    cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
    printf("cycles per dependent load: lds %.1f generic %.1f\n", r[0] / 1e4, r[1] / 1e4);
  }
  return 0;
}
