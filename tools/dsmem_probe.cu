// Development probe (not part of the library): round-trip latency of a 16-B record exchange between
// the two CTAs of a cluster, as the SV loss kernel's row epilogue does once per row.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/dsmem_probe_bin tools/dsmem_probe.cu
// modes: 0 st.shared::cluster + mbarrier.arrive.release.cluster (remote), receiver test_wait.acquire.cluster
//        1 st.async ... mbarrier::complete_tx (receiver arms expect_tx locally)
//        2 same as 0, receiver spins on try_wait (no nanosleep)
//        3 flag polling: st.release.cluster of (value, epoch) into the peer, peer polls ld.acquire.cluster
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) pingpong(int iters, unsigned long long* out) {
  __shared__ __align__(16) float4 rec[2];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ __align__(16) volatile uint32_t flag[4];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const uint32_t peer = rank ^ 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[i])), "r"(1));
    flag[0] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t b = it & 1, ph = (it >> 1) & 1;
      const float v = (float)it;
      if (MODE == 1) {  // arm my barrier for the peer's 16 bytes, then send mine
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(smem_u32(&bar[b])) : "memory");
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%1,%1,%1}, [%2];" ::"r"(
                         mapa(smem_u32(&rec[b]), peer)), "f"(v), "r"(mapa(smem_u32(&bar[b]), peer)) : "memory");
      } else if (MODE == 3) {
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%1,%1,%1};" ::"r"(mapa(smem_u32(&rec[b]), peer)), "f"(v) : "memory");
        asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(mapa(smem_u32((const void*)&flag[0]), peer)), "r"((uint32_t)it + 1) : "memory");
      } else {
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%1,%1,%1};" ::"r"(mapa(smem_u32(&rec[b]), peer)), "f"(v) : "memory");
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(smem_u32(&bar[b]), peer)) : "memory");
      }
      if (MODE == 3) {
        uint32_t f;
        do {
          asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(f) : "r"(smem_u32((const void*)&flag[0])) : "memory");
        } while (f < (uint32_t)it + 1);
      } else {
        uint32_t ok = 0;
        while (!ok) {
          if (MODE == 2)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(smem_u32(&bar[b])), "r"(ph) : "memory");
          else {
            asm volatile("{.reg .pred p; mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(smem_u32(&bar[b])), "r"(ph) : "memory");
            if (!ok) __nanosleep(64);
          }
        }
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(unsigned long long));
  unsigned long long h[296];
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 20000;
  const char* names[] = {"st.shared::cluster + remote arrive, test_wait+sleep", "st.async complete_tx",
                         "st.shared::cluster + remote arrive, try_wait spin", "flag polling (st.release / ld.acquire)"};
  for (int rep = 0; rep < 2; ++rep)
    for (int m = 0; m < 4; ++m) {
      for (int grid : {2, 148}) {
        if (m == 0) pingpong<0><<<grid, 32>>>(iters, d);
        if (m == 1) pingpong<1><<<grid, 32>>>(iters, d);
        if (m == 2) pingpong<2><<<grid, 32>>>(iters, d);
        if (m == 3) pingpong<3><<<grid, 32>>>(iters, d);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("error mode %d\n", m); return 1; }
        cudaMemcpy(h, d, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        if (rep) printf("%-55s grid %3d: %7.1f cycles / exchange (%.0f ns at %d MHz)\n", names[m], grid,
                        mx / iters, mx / iters / (clk / 1e6), clk / 1000);
      }
    }
  return 0;
}
