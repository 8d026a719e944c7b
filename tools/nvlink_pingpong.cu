// NVLink store -> remote poll latency (development probe): GPU 0 and GPU 1 bounce a counter
// through each other's memory (peer access), one thread each; prints the one-way latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pingpong tools/nvlink_pingpong.cu && /tmp/pingpong
#include <cstdio>
#include <cuda_runtime.h>

__global__ void pingpong(volatile unsigned long long* mine, volatile unsigned long long* peer, int first, int iters,
                         unsigned long long* t_out, int weak) {
  const long long t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int i = 0; i < iters; ++i) {
    const unsigned long long want = 2ull * i + (first ? 0 : 1);
    if (!first || i > 0) {
      while (*mine < want) {
      }
    }
    const unsigned long long v = want + 1;
    if (weak)
      asm volatile("st.global.u64 [%0], %1;" ::"l"((unsigned long long*)peer), "l"(v) : "memory");
    else
      *peer = v;
  }
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  t_out[0] = g1 - g0;
  (void)t0;
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("needs 2 GPUs\n"); return 1; }
  unsigned long long *b0, *b1, *t0, *t1;
  cudaSetDevice(0); cudaDeviceEnablePeerAccess(1, 0); cudaMalloc(&b0, 64); cudaMalloc(&t0, 8);
  cudaSetDevice(1); cudaDeviceEnablePeerAccess(0, 0); cudaMalloc(&b1, 64); cudaMalloc(&t1, 8);
  const int iters = 10000;
  for (int weak = 0; weak < 2; ++weak) {
    cudaSetDevice(0); cudaMemset(b0, 0, 64);
    cudaSetDevice(1); cudaMemset(b1, 0, 64);
    cudaDeviceSynchronize(); cudaSetDevice(0); cudaDeviceSynchronize();
    cudaSetDevice(1); pingpong<<<1, 1>>>(b1, b0, 0, iters, t1, weak);
    cudaSetDevice(0); pingpong<<<1, 1>>>(b0, b1, 1, iters, t0, weak);
    cudaDeviceSynchronize(); cudaSetDevice(1); cudaDeviceSynchronize();
    unsigned long long ns = 0;
    cudaSetDevice(0); cudaMemcpy(&ns, t0, 8, cudaMemcpyDeviceToHost);
    printf("%s stores: %d round trips in %.1f us -> one-way store-to-visible latency %.2f us (%s)\n",
           weak ? "weak" : "volatile", iters, ns / 1e3, ns / 1e3 / iters / 2, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
